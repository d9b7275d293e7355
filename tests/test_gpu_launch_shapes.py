"""GPU parity across the launch shapes and internal orders the library can pick.

The create-time tuning knobs (include/mt.h, mt_problem_create) change only how
the work is laid out — which trace mapping runs (chain lanes / ray lanes), the
internal ray order, the deferred-pair queue size, the few-chain multi-block
K3 — never what is computed.  Each shape is checked against the fp64 oracle
with north_star's tolerances, so a layout-specific bug
(a wrong permutation, an overflow path that drops pairs, a buffer sized for the
default shape) fails here even when the default launch is correct.
"""
import contextlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2603_28907_b200 import Problem, inputs  # noqa: E402

DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@contextlib.contextmanager
def env(**kv):
    """Set MT_* knobs for the duration of a mt_problem_create call."""
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def make(prob, max_chains, **knobs):
    with env(**knobs):
        return Problem(prob, device=0, max_chains=max_chains)


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def check_identical_heights(mp, op, H):
    """Path lengths (1e-5 L_tot), log-likelihood (1e-4) and ∂ℓ/∂H (1e-3 rel L2)
    from the same fp32 heights on both sides."""
    Ht = torch.from_numpy(H).to(DEV)
    L_d, _ = mp.path_lengths(Ht)
    ll_d, G_d = mp.loglik_heights(Ht)
    L_o, _ = op.path_lengths(H.astype(np.float64))
    out = op.loglik_grad_H(H.astype(np.float64))
    err = np.abs(L_d.cpu().numpy().astype(np.float64) - L_o).max(2)
    assert np.all(err <= 1e-5 * L_o.sum(2)), float(np.max(err / L_o.sum(2)))
    ll_d, G_d = ll_d.cpu().numpy(), G_d.cpu().numpy().astype(np.float64)
    for c in range(H.shape[0]):
        assert abs(ll_d[c] - out["ll_dev"][c]) <= 1e-4 * abs(out["ll_dev"][c]), c
        assert rel_l2(G_d[c], out["dldH"][c]) <= 1e-3, (c, rel_l2(G_d[c], out["dldH"][c]))


@pytest.mark.parametrize("C,K", [(8, 32), (40, 1), (40, 32), (3, 32)])
def test_both_trace_mappings(problems, oracle_problem, C, K):
    """Chain lanes below their default range (C < 16, ragged 32-chain group) and
    ray lanes above theirs (C = 40 > 16: the per-chain height copies must be
    sized for every chain)."""
    op = oracle_problem("small")
    mp = make(problems("small"), C, MT_TRACE_K=K)
    check_identical_heights(mp, op, inputs.perturbed_heights(op.prob["H_true"], C, 700 + C, scale=1.5))


@pytest.mark.parametrize("C,K", [(2, 1), (33, 32)])
def test_deferred_queue_overflow(problems, oracle_problem, C, K):
    """A one-entry deferred-pair queue: every pair after the first is found through
    the (C x R)-bit redo bitmap by k_trace_defer.  Prior-draw heights (wide band,
    many crossings per ray) defer many pairs in both mappings."""
    op = oracle_problem("small")
    mp = make(problems("small"), C, MT_TRACE_K=K, MT_OVF_CAP=1)
    x = inputs.prior_states("small", C)
    H = np.stack([op.heights(xc.astype(np.float64))[0] for xc in x]).astype(np.float32)
    check_identical_heights(mp, op, H)
    assert mp.trace_counters()["deferred"] > 1


@pytest.mark.parametrize("order", [{"MT_RAY_ORDER": 0}, {"MT_ORDER_Z": 0.9}])
@pytest.mark.parametrize("C", [1, 32])
def test_ray_order_is_invisible(problems, oracle_problem, order, C):
    """Per-ray outputs come back in the caller's ray order whatever the internal
    order: input order and another Morton reference height against the oracle,
    and against the default-order problem ray by ray."""
    op = oracle_problem("small")
    H = inputs.perturbed_heights(op.prob["H_true"], C, 900 + C, scale=1.0)
    mp = make(problems("small"), C, **order)
    check_identical_heights(mp, op, H)
    ref = make(problems("small"), C)
    Ht = torch.from_numpy(H).to(DEV)
    L_a = mp.path_lengths(Ht)[0].cpu().numpy().astype(np.float64)
    L_b = ref.path_lengths(Ht)[0].cpu().numpy().astype(np.float64)
    assert np.all(np.abs(L_a - L_b).max(2) <= 1e-5 * L_b.sum(2))


def test_few_chain_k3_with_and_without_multiblock(problems, oracle_problem):
    """C = 2 < 16: the multi-block K3 (per-chain atomics, last-block finalisation)
    and the one-block-per-chain K3 give the oracle's log-posterior and gradient."""
    op = oracle_problem("small")
    cfg = inputs.CONFIGS["small"]
    x = inputs.chain_states(op.prob["x_true"], 2, cfg.seed + 5)
    out = op.logpost_grad(x.astype(np.float64))
    for knobs in ({}, {"MT_NO_MB": 1}):
        mp = make(problems("small"), 2, **knobs)
        logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
        logp, grad = logp.cpu().numpy(), grad.cpu().numpy().astype(np.float64)
        for c in range(2):
            assert abs(logp[c] - out["logp"][c]) <= 1e-4 * abs(out["logp"][c]), (knobs, c)
            assert rel_l2(grad[c], out["grad"][c]) <= 1e-3, (knobs, c)
