"""Chain sharding end to end on the GPU with two processes:
two ranks on the one available device, gloo for the host-side all-reduces (the
N-GPU bench uses NCCL for the same calls).  No kernel of one rank waits on the
other (chain sharding has no data-path collective), so sharing a device is
only a capacity stand-in.  Each rank runs ChainShard on its contiguous 64 of
128 global chains for 5 warm-up (dual averaging) + 10 sampling iterations.
Every sum of the evaluation is a fixed-point integer sum (R30) and
the trace's launch shape does not depend on the chain count, so every chain's
trajectory, every acceptance and the dual-averaging step size must be
BIT-IDENTICAL to a single-process 128-chain run.  The R-hat all-reduce is
covered with gloo on CPU (test_dist_cpu.py)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, out_dir, n_warm, n_samp):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_28907_b200 import Problem, inputs
    from paper_2603_28907_b200.hmc import ChainShard
    prob = inputs.make_problem("small")
    cfg = inputs.CONFIGS["small"]
    C_total = 128
    C = C_total // world
    off = rank * C
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed, chain_offset=off, super_size=8)
    pb = Problem(prob, device=0, max_chains=C)
    sh = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=10, eps0=cfg.eps, chain_offset=off,
                    n_chains_total=C_total)
    out = sh.run(n_warm, n_samp)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=sh.x.cpu().numpy(), eps=out["eps"],
             acc=np.array(out["warmup_accept"]), acc_prob=sh.acc_prob.cpu().numpy(),
             logp=sh.logp.cpu().numpy(), grad=sh.grad.cpu().numpy(), mean=sh.mean.cpu().numpy(),
             rhat=out["rhat"])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_chain_sharding_matches_one_process(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_2603_28907_b200 import Problem, inputs
    from paper_2603_28907_b200.hmc import ChainShard
    n_warm, n_samp = 5, 10
    port = _free_port()
    mp.spawn(_run, args=(2, port, str(tmp_path), n_warm, n_samp), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"rank{k}.npz") for k in range(2))
    prob = inputs.make_problem("small")
    cfg = inputs.CONFIGS["small"]
    x0 = inputs.chain_states(prob["x_true"], 128, cfg.seed, super_size=8)
    pb = Problem(prob, device=0, max_chains=128)
    sh = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=10, eps0=cfg.eps)
    out = sh.run(n_warm, n_samp)
    # identical all-reduced fixed-point acceptance -> identical dual-averaging step sizes
    assert float(r0["eps"]) == float(r1["eps"]) == out["eps"]
    assert np.array_equal(r0["acc"], r1["acc"]) and np.array_equal(r0["acc"], np.array(out["warmup_accept"]))
    # every chain (global id) followed the same trajectory, bit for bit
    for key, ref in (("x", sh.x), ("acc_prob", sh.acc_prob), ("logp", sh.logp), ("grad", sh.grad),
                     ("mean", sh.mean)):
        both = np.concatenate([r0[key], r1[key]])
        assert np.array_equal(both, ref.cpu().numpy()), key
    # and the all-rank R-hat from the all-reduced partial sums is the single run's
    # (R-hat itself sums fp64 partials over ranks in another order: agreement to rounding)
    np.testing.assert_allclose(r0["rhat"], out["rhat"], rtol=1e-9)


def test_evaluation_is_bit_reproducible_and_independent_of_the_batch():
    """R30: the same chains give bit-identical logp and gradient on repeated
    evaluations and inside larger batches (the 64-chain lane groups are the
    same), including the few-chain and the two-chains-per-lane trace kernels."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_28907_b200 import Problem, inputs
    for name, C in (("small", 256), ("medium", 128)):
        prob = inputs.make_problem(name)
        cfg = inputs.CONFIGS[name]
        x = torch.from_numpy(inputs.chain_states(prob["x_true"], C, cfg.seed)).cuda()
        pb = Problem(prob, device=0, max_chains=C)
        lp1, g1 = pb.logpost_grad(x)
        lp2, g2 = pb.logpost_grad(x)
        assert torch.equal(lp1, lp2) and torch.equal(g1, g2), name
        pb2 = Problem(prob, device=0, max_chains=C // 2)
        lp3, g3 = pb2.logpost_grad(x[C // 2:].contiguous())
        assert torch.equal(lp3, lp1[C // 2:]) and torch.equal(g3, g1[C // 2:]), name
