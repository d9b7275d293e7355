"""Oracle pins for the paper's voxel / sigmoid / linearised forward model
(readings R28/R29 in DESIGN.md).

Pinned against: the ray's in-box extent (Σ_v L_pv = s_exit) and brute-force
point sampling of the voxel map; a vertical ray (n_z pieces of Δz, closed
form); the closed form of λ for a homogeneous density; central finite
differences of the nonlinear λ(R) for G = ∂λ/∂R; the partition of
unity and the γ -> 0 Heaviside limit written as the plain comparisons of
eq:def_LM_density_grid; λ̂ = λ(R0) at the reference geometry; the
second-order error of the linearisation; finite differences of the
full log-posterior.
"""
import numpy as np
import pytest

import oracle
from paper_2603_28907_b200 import inputs

NZ = 20


def _href(prob):
    return np.asarray(prob["H_true"], np.float32).astype(np.float64)


def _edges(X):
    X = np.asarray(X, np.float64)
    return np.concatenate([[X[0]], 0.5 * (X[1:] + X[:-1]), [X[-1]]])


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_voxel_lengths_sum_to_extent(oracle_problem, name):
    op = oracle_problem(name)
    rng = np.random.default_rng(5)
    for q in rng.choice(op.R, 200, replace=False):
        vox, ln = op.voxel_path(NZ, int(q))
        s_exit, _ = op.ray_extent(int(q))
        assert np.all(ln > 0)
        assert np.all((vox >= 0) & (vox < op.N * NZ))
        assert ln.sum() == pytest.approx(s_exit, rel=1e-12)


def test_voxel_lengths_vs_point_sampling(problems, oracle_problem):
    prob = problems("small")
    op = oracle_problem("small")
    ex, ey = _edges(prob["node_x"]), _edges(prob["node_y"])
    dz = float(prob["z_top"]) / NZ
    rng = np.random.default_rng(6)
    M = 200000
    for q in rng.choice(op.R, 12, replace=False):
        q = int(q)
        vox, ln = op.voxel_path(NZ, q)
        s_exit, _ = op.ray_extent(q)
        o = prob["det_xyz"][prob["ray_det"][q]].astype(np.float64)
        d = prob["ray_dir"][q].astype(np.float64)
        h = s_exit / M
        s = (np.arange(M) + 0.5) * h
        p = o[None] + s[:, None] * d[None]
        i = np.clip(np.searchsorted(ex, p[:, 0], side="right") - 1, 0, op.nx - 1)
        j = np.clip(np.searchsorted(ey, p[:, 1], side="right") - 1, 0, op.ny - 1)
        k = np.clip(np.floor(p[:, 2] / dz).astype(int), 0, NZ - 1)
        v = (i * op.ny + j) * NZ + k
        ref = np.bincount(v, minlength=op.N * NZ) * h
        got = np.zeros(op.N * NZ)
        np.add.at(got, vox, ln)
        assert np.max(np.abs(got - ref)) <= 2.5 * h
        assert set(np.flatnonzero(ref)) <= set(vox.tolist()) | set(np.flatnonzero(got))


def test_vertical_ray_closed_form(problems):
    prob = dict(problems("tiny"))
    prob["ray_det"] = np.zeros(1, np.int32)
    prob["ray_dir"] = np.array([[0.0, 0.0, 1.0]], np.float32)
    prob["ray_w"] = np.ones(1, np.float32)
    prob["counts"] = np.ones(1, np.int32)
    op = oracle.Problem(prob)
    vox, ln = op.voxel_path(NZ, 0)
    assert len(vox) == NZ
    assert np.allclose(ln, float(prob["z_top"]) / NZ, rtol=1e-13)
    o = prob["det_xyz"][0]
    i = np.searchsorted(_edges(prob["node_x"]), o[0], side="right") - 1
    j = np.searchsorted(_edges(prob["node_y"]), o[1], side="right") - 1
    assert np.array_equal(vox, (i * op.ny + j) * NZ + np.arange(NZ))


@pytest.mark.parametrize("rho", [0.0, 1.0, 2.65])
def test_lambda_homogeneous_closed_form(problems, oracle_problem, rho):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    lam = op.voxel_lambda(np.full(op.N * NZ, rho), NZ)
    for q in range(0, op.R, 7):
        s_exit, L_ext = op.ray_extent(q)
        ref = float(prob["ray_w"][q]) * np.exp(-(rho * s_exit + prob["rho_ext"] * L_ext) / prob["att_len"])
        assert lam[q] == pytest.approx(ref, rel=1e-13)


def test_G_is_the_gradient_of_lambda(problems, oracle_problem):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    R0 = op.voxel_rhat(_href(prob), NZ)
    rng = np.random.default_rng(7)
    dR = rng.standard_normal(op.N * NZ)
    h = 1e-4
    fd = (op.voxel_lambda(R0 + h * dR, NZ) - op.voxel_lambda(R0 - h * dR, NZ)) / (2 * h)
    lam0 = op.voxel_lambda(R0, NZ)
    for q in range(op.R):
        vox, g, l0 = op.voxel_G_row(R0, NZ, q)
        assert l0 == pytest.approx(lam0[q], rel=1e-14)
        assert np.dot(g, dR[vox]) == pytest.approx(fd[q], rel=1e-7, abs=1e-9 * lam0[q])


def test_rhat_partition_of_unity_and_heaviside_limit(problems, oracle_problem):
    prob = problems("small")
    op = oracle_problem("small")
    H = _href(prob)
    Rh, W = op.voxel_rhat(H, NZ, with_weights=True)
    assert np.allclose(W.sum(0), 1.0, atol=1e-14)
    assert W.min() >= 0.0 and W.max() <= 1.0
    rho = [prob["rho_muck"], prob["rho_air"], prob["rho_rock"]]
    assert Rh.min() >= min(rho) - 1e-12 and Rh.max() <= max(rho) + 1e-12
    # γ -> 0: the Heaviside map of eq:def_LM_density_grid, as plain comparisons
    z = np.arange(NZ) * float(prob["z_top"]) / NZ
    H0 = H[0].reshape(-1)[:, None]
    H1 = H[1].reshape(-1)[:, None]
    ref = np.where(z[None] < H0, rho[0], np.where(z[None] < H1, rho[1], rho[2])).reshape(-1)
    far = (np.abs(z[None] - H0) > 0.05) & (np.abs(z[None] - H1) > 0.05)
    Rs = op.voxel_rhat(H, NZ, gamma=1e-3)
    assert np.allclose(Rs[far.reshape(-1)], ref[far.reshape(-1)], atol=1e-12)
    # z = 0 layer: ς(-0) = 1/2 so the muck indicator at k = 0 is ς(H0) - 1/2 (H_{-1}=0)
    Wt = op.voxel_rhat(H, NZ, gamma=50.0, with_weights=True)[1]
    s = lambda u: 1 / (1 + np.exp(-u / 50.0))  # noqa: E731
    S0 = s(float(prob["z_top"])) - 0.5
    assert np.allclose(Wt[0].reshape(op.N, NZ)[:, 0], (s(H[0].reshape(-1)) - 0.5) / S0, rtol=1e-12)


def _deviance(lam, c):
    c = np.asarray(c, np.float64)
    return np.sum(np.where(c > 0, c * (np.log(lam) - np.log(np.where(c > 0, c, 1.0))), 0.0) - lam + c)


def test_linearised_at_reference_is_exact(problems, oracle_problem):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    x = np.asarray(prob["x_true"], np.float64)[None]
    H = op.heights(x[0])[0]
    out = op.voxel_logpost_grad(x, H, NZ)
    lam = op.voxel_lambda(op.voxel_rhat(H, NZ), NZ)
    assert out["ll_dev"][0] == pytest.approx(_deviance(lam, prob["counts"]), rel=1e-12)
    assert out["prior"][0] == pytest.approx(op.logpost_grad(x)["prior"][0], rel=1e-13)


def test_linearisation_error_is_second_order(problems, oracle_problem):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    Href = _href(prob)
    xr = op.latent_from_heights(Href)
    rng = np.random.default_rng(8)
    dx = rng.standard_normal(op.P)
    err = []
    for t in (1e-4, 2e-4):   # height changes of ~0.05 and ~0.1 m
        x = (xr + t * dx)[None]
        lin = op.voxel_logpost_grad(x, Href, NZ)["ll_dev"][0]
        H = op.heights(x[0])[0]
        full = _deviance(op.voxel_lambda(op.voxel_rhat(H, NZ), NZ), prob["counts"])
        err.append(abs(lin - full))
    assert 3.0 < err[1] / err[0] < 5.0


@pytest.mark.parametrize("href", ["truth", "far"])
def test_voxel_gradient_vs_fd(problems, oracle_problem, href):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    Href = _href(prob)
    if href == "far":   # R0 almost all air: many λ̂ floored (R29)
        Href = np.stack([np.full_like(Href[0], 1.0), np.full_like(Href[1], 299.0)])
    x = inputs.chain_states(prob["x_true"], 2, 1, scale=0.05).astype(np.float64)
    out = op.voxel_logpost_grad(x, Href, NZ)
    assert np.all(np.isfinite(out["logp"])) and np.all(np.isfinite(out["grad"]))
    rng = np.random.default_rng(9)
    for c in range(2):
        for k in rng.choice(op.P, 16, replace=False):
            h = 1e-5
            xp, xm = x.copy(), x.copy()
            xp[c, k] += h
            xm[c, k] -= h
            fd = (op.voxel_logpost_grad(xp[c:c + 1], Href, NZ)["logp"][0]
                  - op.voxel_logpost_grad(xm[c:c + 1], Href, NZ)["logp"][0]) / (2 * h)
            assert out["grad"][c, k] == pytest.approx(fd, rel=2e-5, abs=1e-4)
