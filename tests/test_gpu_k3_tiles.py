"""The group-tiled K3 (k_finish_g: 32-chain groups x 64-node tiles, lane = chain)
on the shapes its indexing has to get right, against the fp64 oracle through
the C ABI (P:532-535 prior stencil on the torus, P:625-642 leapfrog):

  * grids whose node count is below one tile or not a multiple of it, and
    non-square ones, so the x window (n_y halo nodes on each side) wraps the
    torus several times or ends in a partial tile: 3 x 3, 5 x 7, 12 x 12;
  * ragged chain groups (C = 40: one full group of 32 and one of 8);
  * the fused leapfrog's x ping-pong between the caller's block and the second
    buffer at odd and even L (L = 2 ends in the second buffer and copies back);
  * the fp32 Jacobian against round 1's one-block-per-chain K3 (MT_NO_FG=1,
    fp64 Jacobian) on the same inputs.
Tolerances are north_star's: logp 1e-4 relative, gradient 1e-3 relative L2 per
chain; leapfrog per R24b.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs  # noqa: E402

DEV = "cuda:0"


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def grid_problem(base, nx, ny, R=600, seed=5):
    X = inputs.quantize(np.linspace(0.0, 100.0, nx)).astype(np.float32)
    Y = inputs.quantize(np.linspace(0.0, 90.0, ny)).astype(np.float32)
    rng = np.random.default_rng(seed)
    dets = np.concatenate([inputs.quantize(rng.uniform(20, 70, (3, 2))), np.zeros((3, 1))], 1).astype(np.float32)
    th = rng.uniform(0.05, 1.1, R)
    ph = rng.uniform(0, 2 * np.pi, R)
    d = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], 1)
    return dict(base, node_x=X, node_y=Y, det_xyz=dets, ray_det=rng.integers(0, 3, R).astype(np.int32),
                ray_dir=d.astype(np.float32), ray_w=rng.uniform(200, 2000, R).astype(np.float32),
                counts=rng.integers(1, 900, R).astype(np.int32))


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("nx,ny", [(3, 3), (5, 7), (12, 12)])
def test_group_tiled_k3_logpost_and_leapfrog(problems, nx, ny):
    prob = grid_problem(problems("tiny"), nx, ny)
    op = oracle.Problem(prob)
    C, P = 40, 2 * nx * ny
    rng = np.random.default_rng(nx * 100 + ny)
    x0 = (0.4 * rng.standard_normal((C, P))).astype(np.float32)
    mp = Problem(prob, device=0, max_chains=C)
    lp, g = mp.logpost_grad(torch.from_numpy(x0).to(DEV))
    ref = op.logpost_grad(x0.astype(np.float64))
    assert np.allclose(lp.cpu().numpy(), ref["logp"], rtol=1e-4)
    gd = g.cpu().numpy().astype(np.float64)
    for c in range(C):
        assert rel_l2(gd[c], ref["grad"][c]) <= 1e-3, c
    lg = lambda xx: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad(xx))  # noqa: E731
    for L in (2, 3):
        x = torch.from_numpy(x0).to(DEV)
        p = mp.draw_momenta(C, 1234, L)
        p0 = p.cpu().numpy().astype(np.float64)
        logp, grad = mp.logpost_grad(x)
        e = 5e-4
        eps = torch.full((C,), e, dtype=torch.float32, device=DEV)
        mp.leapfrog(x, p, logp, grad, eps, L)
        xo, po, _, _ = oracle.leapfrog(x0.astype(np.float64), p0, e, L, lg)
        xd, pd = x.cpu().numpy().astype(np.float64), p.cpu().numpy().astype(np.float64)
        for c in range(C):
            disp = np.linalg.norm(xo[c] - x0[c])
            bound = 1e-3 * disp + 2 * L * 2.0 ** -24 * np.linalg.norm(x0[c])
            assert np.linalg.norm(xd[c] - xo[c]) <= bound, (L, c)
            assert rel_l2(pd[c], po[c]) <= 1e-3, (L, c)
        # logp / grad returned belong to the final x (in the caller's block)
        r2 = op.logpost_grad(xd)
        assert np.allclose(logp.cpu().numpy(), r2["logp"], rtol=1e-4)


def test_group_tiled_k3_matches_round1_k3(problems):
    """Same inputs through the group-tiled K3 and (MT_NO_FG=1) the one-block-per-chain
    K3 with the fp64 Jacobian: the prior terms are identical operation for operation,
    the chain rule differs by the Jacobian's fp32 rounding only."""
    prob = problems("small")
    cfg = inputs.CONFIGS["small"]
    C = 72
    x = torch.from_numpy(inputs.chain_states(prob["x_true"], C, cfg.seed)).to(DEV)
    lp1, g1 = Problem(prob, device=0, max_chains=C).logpost_grad(x)
    os.environ["MT_NO_FG"] = "1"
    try:
        lp0, g0 = Problem(prob, device=0, max_chains=C).logpost_grad(x)
    finally:
        del os.environ["MT_NO_FG"]
    assert np.allclose(lp1.cpu().numpy(), lp0.cpu().numpy(), rtol=1e-12, atol=1e-6)
    a, b = g1.cpu().numpy().astype(np.float64), g0.cpu().numpy().astype(np.float64)
    for c in range(C):
        assert rel_l2(a[c], b[c]) <= 1e-5, c
