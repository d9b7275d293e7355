"""GPU parity of the non-centred CAR parameterisation (f2, reading
R13d): state (z_0, z_1, ρ_0, ρ_1), x = Q(r)^{-1/2} z applied by a 2-D DFT in
fp64 on the device, against the oracle's direct circulant sums.  Tolerances as
north_star's."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs  # noqa: E402
from test_oracle_ncp import circulant  # noqa: E402

DEV = "cuda:0"


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def ncp_states(prob, op, C, seed, rho=(2.5, 2.0), scale=0.01):
    """z = U(r)^{-1} x for near-posterior centred states x (dense solve, test-side)."""
    x = inputs.chain_states(prob["x_true"], C, seed, scale=scale).astype(np.float64)
    v = np.zeros((C, op.P + 2))
    for l in range(2):
        r = 1.0 / (1.0 + np.exp(-rho[l]))
        U = circulant(oracle.ncp_kernel(op.nx, op.ny, r)[0])
        v[:, l * op.N:(l + 1) * op.N] = np.linalg.solve(U, x[:, l * op.N:(l + 1) * op.N].T).T
        v[:, 2 * op.N + l] = rho[l]
    return v.astype(np.float32)


@pytest.mark.parametrize("name,C,chains", [("tiny", 4, None), ("small", 16, None), ("small", 40, None),
                                           ("medium", 64, [0, 31, 63])])
def test_ncp_logpost_grad(problems, oracle_problem, name, C, chains):
    prob = problems(name)
    op = oracle_problem(name)
    v = ncp_states(prob, op, C, inputs.CONFIGS[name].seed)
    mp = Problem(prob, device=0, max_chains=C, noncentred=True)
    assert mp.P == op.P + 2
    lp, g = mp.logpost_grad(torch.from_numpy(v).to(DEV))
    sel = np.arange(C) if chains is None else np.array(chains)
    ref = op.logpost_grad_ncp(v[sel].astype(np.float64))
    lpd, gd = lp.cpu().numpy(), g.cpu().numpy().astype(np.float64)
    for k, c in enumerate(sel):
        assert abs(lpd[c] - ref["logp"][k]) <= 1e-4 * abs(ref["logp"][k]), (c, lpd[c], ref["logp"][k])
        assert rel_l2(gd[c], ref["grad"][k]) <= 1e-3, (c, rel_l2(gd[c], ref["grad"][k]))
        # the two hyper-parameter components on their own
        assert np.allclose(gd[c, -2:], ref["grad"][k, -2:], rtol=1e-3, atol=1e-3 * np.abs(ref["grad"][k]).max())


def test_ncp_ray_sharded_full_size(problems, oracle_problem):
    """configs[4]: n = 64 (N = 4096 nodes per surface, the 200 KiB shared-memory DFT), 4.19M rays."""
    prob = problems("ray_sharded")
    op = oracle_problem("ray_sharded")
    v = ncp_states(prob, op, 1, inputs.CONFIGS["ray_sharded"].seed)
    mp = Problem(prob, device=0, max_chains=1, noncentred=True)
    lp, g = mp.logpost_grad(torch.from_numpy(v).to(DEV))
    ref = op.logpost_grad_ncp(v.astype(np.float64))
    assert abs(lp[0].item() - ref["logp"][0]) <= 1e-4 * abs(ref["logp"][0])
    assert rel_l2(g[0].cpu().numpy().astype(np.float64), ref["grad"][0]) <= 1e-3


@pytest.mark.parametrize("name,C", [("tiny", 4), ("small", 16)])
def test_ncp_leapfrog_10_steps(problems, oracle_problem, name, C):
    prob = problems(name)
    op = oracle_problem(name)
    v0 = ncp_states(prob, op, C, inputs.CONFIGS[name].seed)
    mp = Problem(prob, device=0, max_chains=C, noncentred=True)
    p0 = np.random.default_rng(12).standard_normal(v0.shape).astype(np.float32)
    e = 2e-4
    x = torch.from_numpy(v0.copy()).to(DEV)
    p = torch.from_numpy(p0.copy()).to(DEV)
    lp, g = mp.logpost_grad(x)
    mp.leapfrog(x, p, lp, g, torch.full((C,), e, dtype=torch.float32, device=DEV), 10)
    lg = lambda vv: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad_ncp(vv))  # noqa: E731
    xo, po, lpo, _ = oracle.leapfrog(v0.astype(np.float64), p0.astype(np.float64), e, 10, lg)
    xd = x.cpu().numpy().astype(np.float64)
    for c in range(C):
        assert rel_l2(xd[c], xo[c]) <= 1e-3, (c, rel_l2(xd[c], xo[c]))
        assert np.linalg.norm(xd[c] - xo[c]) / np.linalg.norm(xo[c] - v0[c]) < 0.05
    ref = op.logpost_grad_ncp(xd)
    assert np.allclose(lp.cpu().numpy(), ref["logp"], rtol=1e-4)


def test_ncp_hmc_step_heights_and_nuts_refusal(problems, oracle_problem):
    prob = problems("small")
    op = oracle_problem("small")
    C = 32
    v = torch.from_numpy(ncp_states(prob, op, C, 2)).to(DEV)
    mp = Problem(prob, device=0, max_chains=C, noncentred=True)
    lp, g = mp.logpost_grad(v)
    eps = torch.full((C,), 2e-4, dtype=torch.float32, device=DEV)
    ap, acc = mp.hmc_step(v, lp, g, eps, 10, seed=11, it=0)
    assert torch.isfinite(lp).all() and torch.isfinite(v).all() and float(ap.mean()) > 0.3
    # logp / grad returned by the step are those of the (accepted or restored) state
    ref = op.logpost_grad_ncp(v.cpu().numpy().astype(np.float64))
    assert np.allclose(lp.cpu().numpy(), ref["logp"], rtol=1e-4)
    # heights of the state are those of x = U z
    H = mp.heights(v[:2]).cpu().numpy().astype(np.float64)
    zz = v[:2].cpu().numpy().astype(np.float64)
    for c in range(2):
        x = np.concatenate([circulant(oracle.ncp_kernel(op.nx, op.ny, 1 / (1 + np.exp(-zz[c, op.P + l])))[0])
                            @ zz[c, l * op.N:(l + 1) * op.N] for l in range(2)])
        sig = [oracle.torus_spectrum(op.nx, op.ny, 1 / (1 + np.exp(-zz[c, op.P + l])))[0] for l in range(2)]
        from scipy.special import ndtr
        u0, u1 = ndtr(x[:op.N] / sig[0]), ndtr(x[op.N:] / sig[1])
        H0 = u0 * op.z_top
        H1 = H0 + u1 * (op.z_top - H0)
        assert np.allclose(H[c].reshape(2, -1), np.stack([H0, H1]), atol=2e-5 * op.z_top)
    from paper_2603_28907_b200 import MTError
    with pytest.raises(MTError):
        mp.nuts_step(v, lp, g, eps, 4, seed=1, it=0)


def test_ncp_ray_shards_sum_to_whole(problems, oracle_problem):
    """Ray sharding (§9) in the non-centred mode: the prior terms (−½|z|², the ρ
    hyperprior) on shard 0 only, the likelihood parts of ∂/∂z and ∂/∂ρ on every
    shard; the partials sum to the unsharded result."""
    prob = problems("small")
    op = oracle_problem("small")
    R = len(prob["ray_det"])
    v = torch.from_numpy(ncp_states(prob, op, 20, 2)).to(DEV)
    whole = Problem(prob, device=0, max_chains=20, noncentred=True)
    lp, g = whole.logpost_grad(v)
    parts = [Problem(prob, device=0, max_chains=20, ray_lo=lo, ray_hi=hi, noncentred=True)
             for lo, hi in ((0, 9000), (9000, R))]
    outs = [p.logpost_grad(v) for p in parts]
    assert np.allclose(sum(o[0].cpu().numpy() for o in outs), lp.cpu().numpy(), rtol=1e-6)
    gsum = sum(o[1].cpu().numpy().astype(np.float64) for o in outs)
    for c in range(20):
        assert rel_l2(gsum[c], g.cpu().numpy()[c].astype(np.float64)) < 1e-5


def test_ncp_non_power_of_two_grid_uses_the_direct_dft(problems):
    """A 12 x 12 grid (not a power of two: the direct-DFT branch of circ_apply,
    the paper's own grids are 19 x 19 / 12 x 15) with zero counts and random z."""
    import dataclasses
    cfg = dataclasses.replace(inputs.CONFIGS["tiny"], name="ncp12", n=12)
    prob = inputs.make_problem(cfg, data={"A": 1.0, "counts": np.zeros(cfg.n_rays, np.int32)})
    op = oracle.Problem(prob)
    C = 3
    rng = np.random.default_rng(5)
    v = np.concatenate([0.3 * rng.standard_normal((C, op.P)), np.tile([[2.0, 1.0]], (C, 1))], axis=1)
    v = v.astype(np.float32)
    mp = Problem(prob, device=0, max_chains=C, noncentred=True)
    lp, g = mp.logpost_grad(torch.from_numpy(v).to(DEV))
    ref = op.logpost_grad_ncp(v.astype(np.float64))
    for c in range(C):
        assert abs(lp[c].item() - ref["logp"][c]) <= 1e-4 * abs(ref["logp"][c])
        assert rel_l2(g[c].cpu().numpy().astype(np.float64), ref["grad"][c]) <= 1e-3


def test_ncp_chain_sharded_8192_bench_launch(problems, oracle_problem):
    """configs[3] in the non-centred mode, the launch `bench.py --noncentred`
    times (8,192 chains), sampled chains."""
    from paper_2603_28907_b200.hmc import noncentred_state
    prob = problems("medium")
    op = oracle_problem("medium")
    cfg = inputs.CONFIGS["chain_sharded"]
    x = inputs.chain_states(prob["x_true"], 8192, cfg.seed, super_size=8)
    rho = np.log(np.asarray(cfg.car_r) / (1.0 - np.asarray(cfg.car_r)))
    v = noncentred_state(x, rho, cfg.n, cfg.n)
    mp = Problem(prob, device=0, max_chains=8192, noncentred=True)
    lp, g = mp.logpost_grad(torch.from_numpy(v).to(DEV))
    sel = np.array([0, 4100, 8191])
    ref = op.logpost_grad_ncp(v[sel].astype(np.float64))
    for k, c in enumerate(sel):
        assert abs(lp[c].item() - ref["logp"][k]) <= 1e-4 * abs(ref["logp"][k])
        assert rel_l2(g[c].cpu().numpy().astype(np.float64), ref["grad"][k]) <= 1e-3


def test_ncp_with_the_voxel_model(problems, oracle_problem):
    """Non-centred (f2) × voxel model (f3): with ρ = logit(car_r) the copula scale
    σ(r) is the fixed-r one, so the voxel oracle at x = U z gives the likelihood;
    logp = ll − ½|z|² − N ln 2π + Σ ln r(1−r) and ∂/∂z = −z + U ∂ll/∂x."""
    from test_oracle_prior import dense_Q
    prob = problems("tiny")
    op = oracle_problem("tiny")
    cfg = inputs.CONFIGS["tiny"]
    r = cfg.car_r[0]
    rho = np.log(r / (1 - r))
    C = 3
    v = ncp_states(prob, op, C, cfg.seed, rho=(rho, rho))
    mp = Problem(prob, device=0, max_chains=C, noncentred=True)
    Hr = np.asarray(prob["H_true"], np.float32)
    mp.voxel_model(60, Hr)
    lp, g = mp.logpost_grad(torch.from_numpy(v).to(DEV))
    U = circulant(oracle.ncp_kernel(op.nx, op.ny, r)[0])
    Q = dense_Q(op.nx, op.ny, r)
    for c in range(C):
        z = v[c, :op.P].astype(np.float64)
        x = np.concatenate([U @ z[:op.N], U @ z[op.N:]])
        o = op.voxel_logpost_grad(x[None], Hr.astype(np.float64), 60)
        gx_ll = o["grad"][0] + np.concatenate([Q @ x[:op.N], Q @ x[op.N:]])   # remove the centred prior
        ref_lp = o["ll_dev"][0] - 0.5 * z @ z - op.N * np.log(2 * np.pi) + 2 * np.log(r * (1 - r))
        ref_gz = -z + np.concatenate([U @ gx_ll[:op.N], U @ gx_ll[op.N:]])
        assert abs(lp[c].item() - ref_lp) <= 1e-4 * abs(ref_lp)
        assert rel_l2(g[c, :op.P].cpu().numpy().astype(np.float64), ref_gz) <= 1e-3


@pytest.mark.parametrize("rho", [(-3.0, 6.0), (0.0, -1.0)])
def test_ncp_extreme_dependence(problems, oracle_problem, rho):
    """r_l = logistic(ρ_l) from 0.047 (nearly independent nodes) to 0.9975
    (λ_min = 4 − 4r ≈ 0.01: the circulant's largest eigenvalue ≈ 100)."""
    prob = problems("tiny")
    op = oracle_problem("tiny")
    C = 3
    rng = np.random.default_rng(9)
    v = np.concatenate([0.3 * rng.standard_normal((C, op.P)), np.tile([list(rho)], (C, 1))], axis=1)
    v = v.astype(np.float32)
    mp = Problem(prob, device=0, max_chains=C, noncentred=True)
    lp, g = mp.logpost_grad(torch.from_numpy(v).to(DEV))
    ref = op.logpost_grad_ncp(v.astype(np.float64))
    for c in range(C):
        assert abs(lp[c].item() - ref["logp"][c]) <= 1e-4 * abs(ref["logp"][c])
        assert rel_l2(g[c].cpu().numpy().astype(np.float64), ref["grad"][c]) <= 1e-3
