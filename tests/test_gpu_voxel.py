"""GPU parity of the paper's voxel / sigmoid / linearised forward model (f3,
P:242-390; readings R28/R29) through the C ABI (mt_voxel_model + the usual
evaluation entry points) against the fp64 oracle (oracle.Problem.voxel_*).

Tolerances are north_star's: logp 1e-4 relative per chain,
gradient 1e-3 relative L2 per chain, 10 leapfrog steps 1e-3 relative L2; the
non-zero count of G is an integer and must match exactly.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs  # noqa: E402

DEV = "cuda:0"
NZ = 60


def href(prob):
    return np.asarray(prob["H_true"], np.float32)


@pytest.fixture(scope="module")
def vgpu(problems):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cache = {}

    def get(name, max_chains=None):
        key = (name, max_chains)
        if key not in cache:
            cfg = inputs.CONFIGS[name]
            mp = Problem(problems(name), device=0, max_chains=max_chains or cfg.chains)
            mp.voxel_model(NZ, href(problems(name)))
            cache[key] = mp
        return cache[key]
    return get


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def check(op, prob, x, chains, logp_d, grad_d):
    out = op.voxel_logpost_grad(x[chains].astype(np.float64), href(prob).astype(np.float64), NZ)
    fails = []
    for k, c in enumerate(chains):
        e_lp = abs(logp_d[c] - out["logp"][k]) / abs(out["logp"][k])
        e_g = rel_l2(grad_d[c].astype(np.float64), out["grad"][k])
        if not (e_lp <= 1e-4 and e_g <= 1e-3):
            fails.append((int(c), e_lp, e_g))
    return fails


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_voxel_nnz_matches_oracle(vgpu, oracle_problem, name):
    mp, op = vgpu(name), oracle_problem(name)
    info = mp.voxel_info()
    assert info["n_z"] == NZ and info["n_grid"] == op.N * NZ
    assert info["nnz"] == sum(len(op.voxel_path(NZ, q)[0]) for q in range(op.R))


@pytest.mark.parametrize("name,C", [("tiny", 4), ("small", 8), ("small", 17), ("small", 64)])
def test_voxel_logpost_grad(vgpu, oracle_problem, problems, name, C):
    """Row lanes (C < 16) and chain lanes (C >= 16, a ragged group at 17)."""
    prob = problems(name)
    mp, op = vgpu(name, max_chains=64 if name == "small" else None), oracle_problem(name)
    x = inputs.chain_states(prob["x_true"], C, inputs.CONFIGS[name].seed, scale=0.05)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    fails = check(op, prob, x, np.arange(C), logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


def test_voxel_medium_bench_launch(vgpu, oracle_problem, problems):
    """Full Medium size in the launch configuration bench.py --model voxel times
    (1024 chains), sampled chains."""
    prob = problems("medium")
    mp, op = vgpu("medium"), oracle_problem("medium")
    x = inputs.chain_states(prob["x_true"], 1024, inputs.CONFIGS["medium"].seed)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    fails = check(op, prob, x, np.array([0, 511, 1023]), logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


def test_voxel_ray_sharded_full_size(vgpu, oracle_problem, problems):
    """configs[4] at full size (4,194,304 rays, 64x64x60 voxels), one chain (row lanes)."""
    prob = problems("ray_sharded")
    mp, op = vgpu("ray_sharded"), oracle_problem("ray_sharded")
    x = inputs.chain_states(prob["x_true"], 1, inputs.CONFIGS["ray_sharded"].seed)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    fails = check(op, prob, x, np.array([0]), logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


def test_voxel_far_reference_floors(problems, oracle_problem):
    """R0 almost all air: many λ̂ hit the R29 floor; GPU and oracle agree."""
    prob = problems("tiny")
    op = oracle_problem("tiny")
    mp = Problem(prob, device=0, max_chains=4)
    Hf = np.stack([np.full((op.nx, op.ny), 1.0), np.full((op.nx, op.ny), 299.0)]).astype(np.float32)
    mp.voxel_model(NZ, Hf)
    x = inputs.chain_states(prob["x_true"], 4, 1, scale=0.05)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    out = op.voxel_logpost_grad(x.astype(np.float64), Hf.astype(np.float64), NZ)
    for c in range(4):
        assert abs(logp[c].item() - out["logp"][c]) <= 1e-4 * abs(out["logp"][c])
        assert rel_l2(grad[c].cpu().numpy().astype(np.float64), out["grad"][c]) <= 1e-3


@pytest.mark.parametrize("name,C", [("tiny", 4), ("small", 16)])
def test_voxel_leapfrog_10_steps(vgpu, oracle_problem, problems, name, C):
    prob = problems(name)
    mp, op = vgpu(name, max_chains=64 if name == "small" else None), oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    Hr = href(prob).astype(np.float64)
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
    p0 = np.random.default_rng(11).standard_normal(x0.shape).astype(np.float32)
    eps = np.full(C, cfg.eps, np.float32)
    xd = torch.from_numpy(x0.copy()).to(DEV)
    pd = torch.from_numpy(p0.copy()).to(DEV)
    lp, g = mp.logpost_grad(xd)
    mp.leapfrog(xd, pd, lp, g, torch.from_numpy(eps).to(DEV), 10)

    def lg(x):
        o = op.voxel_logpost_grad(x, Hr, NZ)
        return o["logp"], o["grad"]
    xo, po, lpo, _ = oracle.leapfrog(x0.astype(np.float64), p0.astype(np.float64), eps.astype(np.float64), 10, lg)
    xf = xd.cpu().numpy().astype(np.float64)
    for c in range(C):
        assert rel_l2(xf[c], xo[c]) <= 1e-3, (c, rel_l2(xf[c], xo[c]))   # north_star criterion
        assert np.linalg.norm(xf[c] - xo[c]) / np.linalg.norm(xo[c] - x0[c]) < 0.05
    # the fused leapfrog's logp / grad are those of its own final x
    ref = op.voxel_logpost_grad(xf, Hr, NZ)
    assert np.allclose(lp.cpu().numpy(), ref["logp"], rtol=1e-4)
    for c in range(C):
        assert rel_l2(g.cpu().numpy()[c].astype(np.float64), ref["grad"][c]) <= 1e-3


def test_voxel_hmc_step_and_switch_back(problems):
    """One HMC step under the voxel model runs and stays finite; n_z = 0 restores
    the exact model (up to the exact tracer's atomic summation order)."""
    prob = problems("small")
    cfg = inputs.CONFIGS["small"]
    x = torch.from_numpy(inputs.chain_states(prob["x_true"], 32, cfg.seed)).to(DEV)
    mp = Problem(prob, device=0, max_chains=32)
    lp_exact, g_exact = mp.logpost_grad(x)
    mp.voxel_model(NZ, href(prob))
    xs = x.clone()
    lp, g = mp.logpost_grad(xs)
    eps = torch.full((32,), cfg.eps, dtype=torch.float32, device=DEV)
    out = mp.hmc_step(xs, lp, g, eps, 10, seed=7, it=0)
    assert torch.isfinite(lp).all() and torch.isfinite(xs).all()
    assert 0.0 <= float(out[0].float().mean()) <= 1.0
    mp.voxel_model(0)
    assert mp.voxel_info()["n_z"] == 0
    lp2, g2 = mp.logpost_grad(x)
    assert torch.allclose(lp2, lp_exact, rtol=1e-9, atol=0)
    assert float((g2 - g_exact).norm() / g_exact.norm()) < 1e-5


def test_voxel_ray_shards_sum_to_whole(problems):
    """Ray sharding (§9) under the voxel model: each shard's problem builds G for
    its rays; partial logp / grad (prior on shard 0) sum to the unsharded result."""
    prob = problems("small")
    R = len(prob["ray_det"])
    cfg = inputs.CONFIGS["small"]
    x = torch.from_numpy(inputs.chain_states(prob["x_true"], 40, cfg.seed)).to(DEV)
    whole = Problem(prob, device=0, max_chains=40)
    whole.voxel_model(NZ, href(prob))
    lp, g = whole.logpost_grad(x)
    lps, gs = [], []
    for lo, hi in ((0, 7000), (7000, R)):
        part = Problem(prob, device=0, max_chains=40, ray_lo=lo, ray_hi=hi)
        part.voxel_model(NZ, href(prob))
        a, b = part.logpost_grad(x)
        lps.append(a.cpu().numpy())
        gs.append(b.cpu().numpy().astype(np.float64))
    assert np.allclose(sum(lps), lp.cpu().numpy(), rtol=1e-6)
    gsum = sum(gs)
    for c in range(40):
        assert rel_l2(gsum[c], g.cpu().numpy()[c].astype(np.float64)) < 1e-5


def test_voxel_nuts_step_matches_oracle(vgpu, oracle_problem, problems):
    """The batched NUTS transition (f1) on the voxel model (f3): same Philox
    streams as the oracle's NUTS driven by the voxel oracle; trees of <= 16 leaves."""
    prob = problems("tiny")
    mp, op = vgpu("tiny"), oracle_problem("tiny")
    cfg = inputs.CONFIGS["tiny"]
    Hr = href(prob).astype(np.float64)
    C, max_depth, e, seed, it = 4, 4, 2e-3, inputs.philox_key(cfg), 5
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
    x = torch.from_numpy(x0).to(DEV)
    lp, g = mp.logpost_grad(x)
    eps = torch.full((C,), e, dtype=torch.float32, device=DEV)
    acc, depth, nl = mp.nuts_step(x, lp, g, eps, max_depth, seed, it)
    xd = x.cpu().numpy().astype(np.float64)
    lg1 = lambda th: (lambda o: (o["logp"][0], o["grad"][0]))(op.voxel_logpost_grad(th[None], Hr, NZ))  # noqa: E731
    agree = 0
    for c in range(C):
        lp0, g0 = lg1(x0[c].astype(np.float64))
        ref = oracle.nuts_step(x0[c], lp0, g0, e, lg1, seed, it, c, max_depth=max_depth)
        if ref["depth"] == depth[c].item() and ref["n_leaves"] == nl[c].item():
            agree += 1
            assert rel_l2(xd[c], ref["x"]) <= 1e-3
    assert agree >= C - 1, agree


def test_voxel_chain_sharded_8192_bench_launch(oracle_problem, problems):
    """configs[3] under the voxel model in the launch configuration
    `bench.py --model voxel` times (8,192 chains, 4 per lane), sampled chains."""
    prob = problems("medium")
    op = oracle_problem("medium")
    mp = Problem(prob, device=0, max_chains=8192)
    mp.voxel_model(NZ, href(prob))
    x = inputs.chain_states(prob["x_true"], 8192, inputs.CONFIGS["chain_sharded"].seed, super_size=8)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    fails = check(op, prob, x, np.array([0, 4095, 8191]), logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


@pytest.mark.parametrize("nz,gamma", [(1, 1.0), (7, 0.2), (200, 1.0), (60, 8.0)])
def test_voxel_edge_grids_and_sigmoid_scales(problems, oracle_problem, nz, gamma):
    """Degenerate and extreme voxel grids (one layer; 1.5 m layers) and sigmoid
    scales (γ = 0.2 m: nearly Heaviside; 8 m: very smooth) against the oracle."""
    prob = problems("tiny")
    op = oracle_problem("tiny")
    Hr = href(prob)
    mp = Problem(prob, device=0, max_chains=4)
    mp.voxel_model(nz, Hr, gamma=gamma)
    x = inputs.chain_states(prob["x_true"], 4, 1, scale=0.05)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    out = op.voxel_logpost_grad(x.astype(np.float64), Hr.astype(np.float64), nz, gamma=gamma)
    for c in range(4):
        assert abs(logp[c].item() - out["logp"][c]) <= 1e-4 * abs(out["logp"][c]), (c, nz, gamma)
        assert rel_l2(grad[c].cpu().numpy().astype(np.float64), out["grad"][c]) <= 1e-3, (c, nz, gamma)
