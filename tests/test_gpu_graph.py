"""CUDA-graph replay of the sampling step (ChainShard.step_graph, mt_set_step_counters)
against eager stepping: the Philox iteration (R22) and the Welford count live on the
device and advance inside the captured step, so every replay is the next HMC
iteration — and, every sum being order-independent (R30), the chains'
states, log-posteriors, gradients, acceptance statistics and Welford moments must
equal the eager run's bit for bit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2603_28907_b200 import Problem, inputs  # noqa: E402
from paper_2603_28907_b200.hmc import ChainShard  # noqa: E402


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name,C", [("small", 64), ("medium", 128)])
def test_graph_replay_equals_eager_steps(problems, name, C):
    prob = problems(name)
    cfg = inputs.CONFIGS[name]
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
    shards = []
    for mode in ("eager", "graph"):
        pb = Problem(prob, device=0, max_chains=C)
        sh = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=10, eps0=cfg.eps)
        sh.step(adapt=False, sample=True, monitor=True)   # one eager step (the graph path's first, too)
        for k in range(6):
            if mode == "eager":
                sh.step(adapt=False, sample=True, monitor=True)
            else:
                sh.step_graph(sample=True, monitor=True)
        torch.cuda.synchronize()
        shards.append(sh)
    a, b = shards
    assert a.it == b.it and a.n_samples == b.n_samples
    assert int(b._it_dev.item()) == b.it and int(b._n_dev.item()) == b.n_samples
    for key in ("x", "logp", "grad", "acc_prob", "accepted", "mean", "m2", "acc_mon"):
        assert torch.equal(getattr(a, key), getattr(b, key)), key
    assert b.launches_per_graph_step > 4 * 10
    # an eager step after graph replays continues from the device counters
    a.step(adapt=False, sample=True, monitor=True)
    b.step(adapt=False, sample=True, monitor=True)
    for key in ("x", "logp", "mean", "m2"):
        assert torch.equal(getattr(a, key), getattr(b, key)), key


def test_step_counters_replace_the_host_arguments(problems):
    """With device counters set, mt_hmc_step ignores its host iteration and
    mt_stats_update its host count (and both advance the device values)."""
    prob = problems("tiny")
    cfg = inputs.CONFIGS["tiny"]
    C = 4
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
    out = []
    for use_dev in (False, True):
        pb = Problem(prob, device=0, max_chains=C)
        x = torch.from_numpy(x0).cuda()
        lp, g = pb.logpost_grad(x)
        eps = torch.full((C,), cfg.eps, dtype=torch.float32, device="cuda")
        mean = torch.zeros_like(x)
        m2 = torch.zeros_like(x)
        it_d = torch.tensor([7], dtype=torch.int64, device="cuda")
        n_d = torch.tensor([3], dtype=torch.int32, device="cuda")
        if use_dev:
            pb.set_step_counters(it_d, n_d)
        ap, acc = pb.hmc_step(x, lp, g, eps, 5, inputs.philox_key(cfg), 12345 if use_dev else 7)
        pb.stats_update(C, x=x, n_prev=99 if use_dev else 3, mean=mean, m2=m2)
        torch.cuda.synchronize()
        if use_dev:
            assert int(it_d.item()) == 8 and int(n_d.item()) == 4
            pb.set_step_counters(None, None)
        out.append((x.clone(), lp.clone(), ap.clone(), mean.clone(), m2.clone()))
    for u, v in zip(*out):
        assert torch.equal(u, v)
