"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Tolerances are BASELINE.json north_star's, read as in
DESIGN.md "Tolerances":
  traversal   bit-exact (i, j) lists
  lengths     |L_dev - L_ora| <= 1e-5 * L_tot per (chain, ray, unit)
  logpost     |Δ| <= 1e-4 |logp_ora| per chain (deviance-centred form + prior)
  gradient    ||Δ||_2 <= 1e-3 ||g_ora||_2 per chain
  leapfrog    ||x10_dev - x10_ora||_2 <= 1e-3 ||x10_ora||_2 per chain (north_star as written)
              and, displacement-relative (R24b),
              ||x10_dev - x10_ora||_2 <= 1e-3 ||x10_ora - x0||_2 + 2 L 2^-24 ||x0||_2
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs, philox  # noqa: E402

DEV = "cuda:0"


@pytest.fixture(scope="module")
def gpu(problems):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cache = {}

    def get(name, max_chains=None, **kw):
        key = (name, max_chains, tuple(sorted(kw.items())))
        if key not in cache:
            cfg = inputs.CONFIGS[name]
            cache[key] = Problem(problems(name), device=0, max_chains=max_chains or cfg.chains, **kw)
        return cache[key]
    return get


def _record_margin(key, value):
    import json
    import os
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, "parity_margins.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[key] = value
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def sampling_eps(name):
    """The sampling-phase step size (tools/tune_eps.py) when tuned, else the config's."""
    import json
    import os
    path = os.path.join(inputs.DATA_DIR, "tuned_eps.json")
    tuned = json.load(open(path)) if os.path.exists(path) else {}
    return tuned.get(name, {}).get("eps", inputs.CONFIGS[name].eps)


# ---------------------------------------------------------------------------
# traversal (integer, bit-exact)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,nsample", [("tiny", None), ("small", 3000), ("medium", 2000),
                                          ("ray_sharded", 1500)])
def test_traversal_bit_exact(gpu, oracle_problem, name, nsample):
    mp, op = gpu(name), oracle_problem(name)
    rays = range(op.R) if nsample is None else np.random.default_rng(7).choice(op.R, nsample, replace=False)
    for q in rays:
        q = int(q)
        ij_d, si_d, so_d = mp.debug_traversal(q)
        ij_o, si_o, so_o = op.traversal(q)
        assert np.array_equal(ij_d, ij_o), q
        assert np.allclose(so_d, so_o, rtol=2e-6, atol=1e-5), q


# ---------------------------------------------------------------------------
# path lengths and likelihood/adjoint from identical heights
# ---------------------------------------------------------------------------
def identical_heights(prob, C, seed, scale=2.0):
    return inputs.perturbed_heights(prob["H_true"], C, seed, scale=scale)


@pytest.mark.parametrize("name,C", [("tiny", 4), ("small", 8), ("medium", 2), ("ray_sharded", 1)])
def test_path_lengths_identical_heights(gpu, oracle_problem, name, C):
    mp, op = gpu(name), oracle_problem(name)
    H = identical_heights(op.prob, C, 100 + C)
    L_d, O_d = mp.path_lengths(torch.from_numpy(H).to(DEV))
    L_o, O_o = op.path_lengths(H.astype(np.float64))
    Ltot = L_o.sum(2)
    err = np.abs(L_d.cpu().numpy().astype(np.float64) - L_o).max(2)
    bad = err > 1e-5 * Ltot
    assert bad.sum() == 0, f"{bad.sum()} of {bad.size} (chain, ray) pairs exceed 1e-5 L_tot; max rel {np.max(err / Ltot):.3g}"
    assert np.allclose(O_d.cpu().numpy(), O_o, rtol=2e-5)


@pytest.mark.parametrize("name,C", [("tiny", 4), ("small", 8), ("medium", 2), ("ray_sharded", 1)])
def test_loglik_and_adjoint_identical_heights(gpu, oracle_problem, name, C):
    mp, op = gpu(name), oracle_problem(name)
    H = identical_heights(op.prob, C, 200 + C, scale=1.0)
    ll_d, G_d = mp.loglik_heights(torch.from_numpy(H).to(DEV))
    out = op.loglik_grad_H(H.astype(np.float64))
    ll_d = ll_d.cpu().numpy()
    G_d = G_d.cpu().numpy().astype(np.float64)
    for c in range(C):
        assert abs(ll_d[c] - out["ll_dev"][c]) <= 1e-4 * abs(out["ll_dev"][c]), (c, ll_d[c], out["ll_dev"][c])
        assert rel_l2(G_d[c], out["dldH"][c]) <= 1e-3, (c, rel_l2(G_d[c], out["dldH"][c]))


def test_caller_heights_at_full_chain_count(gpu, oracle_problem):
    """mt_path_lengths / mt_loglik_heights with C = max_chains (64): every workspace
    clear covers whole 32-chain groups (a precedence bug once cleared too much)."""
    mp, op = gpu("small"), oracle_problem("small")
    C = mp.max_chains
    H = identical_heights(op.prob, C, 300, scale=1.0)
    L_d, _ = mp.path_lengths(torch.from_numpy(H).to(DEV))
    ll_d, G_d = mp.loglik_heights(torch.from_numpy(H).to(DEV))
    sel = [0, 31, 32, C - 1]
    L_o, _ = op.path_lengths(H[sel].astype(np.float64))
    out = op.loglik_grad_H(H[sel].astype(np.float64))
    L_d = L_d.cpu().numpy()[sel].astype(np.float64)
    assert np.all(np.abs(L_d - L_o).max(2) <= 1e-5 * L_o.sum(2))
    for k, c in enumerate(sel):
        assert abs(ll_d.cpu().numpy()[c] - out["ll_dev"][k]) <= 1e-4 * abs(out["ll_dev"][k])
        assert rel_l2(G_d.cpu().numpy()[c].astype(np.float64), out["dldH"][k]) <= 1e-3


def test_heights_map(gpu, oracle_problem):
    mp, op = gpu("small"), oracle_problem("small")
    x = inputs.chain_states(op.prob["x_true"], 8, 2, scale=0.3)
    H_d = mp.heights(torch.from_numpy(x).to(DEV)).cpu().numpy()
    H_o = np.stack([op.heights(xc.astype(np.float64))[0] for xc in x])
    # fp64 internally, one fp32 rounding at the end
    assert np.allclose(H_d, H_o, rtol=1.5 * 2 ** -24, atol=0)


# ---------------------------------------------------------------------------
# end-to-end log-posterior and gradient from x
# ---------------------------------------------------------------------------
def e2e_check(mp, op, x, chains, logp_d, grad_d):
    out = op.logpost_grad(x[chains].astype(np.float64))
    fails = []
    for k, c in enumerate(chains):
        e_lp = abs(logp_d[c] - out["logp"][k]) / abs(out["logp"][k])
        e_g = rel_l2(grad_d[c].astype(np.float64), out["grad"][k])
        if e_lp > 1e-4 or e_g > 1e-3:
            fails.append((int(c), e_lp, e_g))
    return fails


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_logpost_grad_end_to_end(gpu, oracle_problem, name):
    mp, op = gpu(name), oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    x = inputs.chain_states(op.prob["x_true"], cfg.chains, cfg.seed)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    fails = e2e_check(mp, op, x, np.arange(cfg.chains), logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


def test_logpost_grad_ray_sharded_full_size(gpu, oracle_problem):
    """configs[4] at full size (4,194,304 rays, 8,192 params, one chain): the
    single-chain ray-lanes path.  This chain has crossings with |g'| ~ 1e-5, where
    ∇ₓ moves by 1.2e-2 (relative) between fp64 and fp32-rounded heights
    (tools/e2e_diag.py): the fp64 re-solves must use the fp64 heights (HP2)."""
    mp, op = gpu("ray_sharded"), oracle_problem("ray_sharded")
    cfg = inputs.CONFIGS["ray_sharded"]
    x = inputs.chain_states(op.prob["x_true"], cfg.chains, cfg.seed)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    fails = e2e_check(mp, op, x, np.array([0]), logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


def test_logpost_grad_chain_sharded_8192(gpu, oracle_problem):
    """configs[3] in the launch configuration bench.py times at N = 1: all 8,192
    chains (super-chains of 8 share a start) on one device, compared on sampled
    chains the oracle computes one by one."""
    mp, op = gpu("medium", max_chains=8192), oracle_problem("medium")
    cfg = inputs.CONFIGS["chain_sharded"]
    x = inputs.chain_states(op.prob["x_true"], 8192, cfg.seed, super_size=8)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    chains = np.array([0, 4095, 4100, 8191])
    fails = e2e_check(mp, op, x, chains, logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


@pytest.mark.parametrize("name,C,chains", [("small", 64, None), ("medium", 1024, [0, 77, 1023])])
def test_logpost_grad_prior_draw_states(gpu, oracle_problem, name, C, chains):
    """The wide-band "prior-draw" chain states: heights spread over
    the whole box, every in-box cell in the band, many crossings per ray."""
    mp, op = gpu(name), oracle_problem(name)
    x = inputs.prior_states(name, C)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    sel = np.arange(C) if chains is None else np.array(chains)
    fails = e2e_check(mp, op, x, sel, logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


def test_logpost_grad_medium_bench_launch(gpu, oracle_problem):
    """Full Medium size, in the launch configuration bench.py times (1024 chains),
    compared on sampled chains the oracle computes one by one."""
    mp, op = gpu("medium"), oracle_problem("medium")
    cfg = inputs.CONFIGS["medium"]
    x = inputs.chain_states(op.prob["x_true"], cfg.chains, cfg.seed)
    logp, grad = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    chains = np.array([0, 511, 1023])
    fails = e2e_check(mp, op, x, chains, logp.cpu().numpy(), grad.cpu().numpy())
    assert not fails, fails


# ---------------------------------------------------------------------------
# momenta, leapfrog, HMC
# ---------------------------------------------------------------------------
def test_philox_bit_exact_vs_oracle_and_curand(gpu):
    rng = np.random.default_rng(3)
    ctr = rng.integers(0, 2 ** 32, size=(4096, 4), dtype=np.uint64).astype(np.uint32)
    key = [int(v) for v in rng.integers(0, 2 ** 32, size=2, dtype=np.uint64)]
    c = torch.from_numpy(ctr.view(np.int32)).to(DEV)
    d = philox(c, key).cpu().numpy().view(np.uint32)
    cu = philox(c, key, use_curand=True).cpu().numpy().view(np.uint32)
    assert np.array_equal(d, cu)
    for k in range(0, 4096, 97):
        assert np.array_equal(d[k], oracle.philox4x32_10(ctr[k], key))


def test_momenta_match_oracle(gpu, oracle_problem):
    mp = gpu("small")
    P = mp.P
    seed, it, off = 0xDEADBEEF12345678, 17, 40
    p_d = mp.draw_momenta(8, seed, it, off).cpu().numpy()
    for c in range(8):
        assert np.allclose(p_d[c], oracle.momenta(P, seed, it, off + c), rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("name,C", [("tiny", 4), ("small", 16), ("medium", 2), ("ray_sharded", 1)])
def test_leapfrog_10_steps(gpu, oracle_problem, name, C):
    mp, op = gpu(name), oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    x0 = inputs.chain_states(op.prob["x_true"], C, cfg.seed)
    seed = inputs.philox_key(cfg)
    x = torch.from_numpy(x0).to(DEV)
    p = mp.draw_momenta(C, seed, 0)
    p0 = p.cpu().numpy().astype(np.float64)
    logp, grad = mp.logpost_grad(x)
    e = sampling_eps(name)
    eps = torch.full((C,), e, dtype=torch.float32, device=DEV)
    mp.leapfrog(x, p, logp, grad, eps, 10)
    xo, po, lpo, go = oracle.leapfrog(x0.astype(np.float64), p0, e, 10,
                                      lambda xx: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad(xx)))
    xd = x.cpu().numpy().astype(np.float64)
    worst = 0.0
    for c in range(C):
        assert rel_l2(xd[c], xo[c]) <= 1e-3, (c, rel_l2(xd[c], xo[c]))   # north_star criterion as written
        # displacement-relative (R24b): 1e-3 of the oracle's own displacement, plus the fp32 floor of
        # the state block (each of the L drifts rounds x once: <= 2^-24 ||x|| per step; factor 2 for
        # the momentum and gradient roundings it feeds)
        disp = np.linalg.norm(xo[c] - x0[c])
        bound = 1e-3 * disp + 2 * 10 * 2.0 ** -24 * np.linalg.norm(x0[c])
        err = np.linalg.norm(xd[c] - xo[c])
        worst = max(worst, err / bound)
        assert err <= bound, (c, err, disp, bound)
    _record_margin(f"leapfrog10/{name}", worst)
    # logp/grad returned by the fused leapfrog are those of its own final x.  (Comparing with
    # the oracle's trajectory end instead is ill-conditioned: |∇logp| ~ 1e5, so position
    # differences well inside 1e-3 move logp by O(10).)
    ref = op.logpost_grad(xd)
    assert np.allclose(logp.cpu().numpy(), ref["logp"], rtol=1e-4)
    for c in range(C):
        assert rel_l2(grad.cpu().numpy()[c].astype(np.float64), ref["grad"][c]) <= 1e-3


def test_hmc_step_matches_oracle_decisions(gpu, oracle_problem):
    name, C = "small", 16
    mp, op = gpu(name), oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    x0 = inputs.chain_states(op.prob["x_true"], C, cfg.seed)
    seed = inputs.philox_key(cfg)
    x = torch.from_numpy(x0).to(DEV)
    logp, grad = mp.logpost_grad(x)
    e = sampling_eps(name)
    eps = torch.full((C,), e, dtype=torch.float32, device=DEV)
    ap, acc = mp.hmc_step(x, logp, grad, eps, 10, seed, 3)
    lg = lambda xx: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad(xx))  # noqa: E731
    xo, apo, acco, lpo, dHo = oracle.hmc_step(x0.astype(np.float64), e, 10, lg, seed, 3)
    u = np.array([oracle.mh_uniform(seed, 3, c) for c in range(C)])
    clear = np.abs(np.log(u) + dHo) > 0.05      # decisions far from the threshold must agree
    acc = acc.cpu().numpy().astype(bool)
    assert clear.sum() >= C // 2
    assert np.array_equal(acc[clear], acco[clear])
    assert np.allclose(ap.cpu().numpy()[clear], apo[clear], atol=0.02)
    xd = x.cpu().numpy()
    for c in np.nonzero(clear)[0]:
        assert rel_l2(xd[c], xo[c]) <= 1e-3


# ---------------------------------------------------------------------------
# edge cases
# ---------------------------------------------------------------------------
def test_zero_chains_and_bad_arguments(gpu):
    from paper_2603_28907_b200 import MTError
    mp = gpu("tiny")
    x = torch.zeros((0, mp.P), device=DEV)
    lp, g = mp.logpost_grad(x)
    assert lp.numel() == 0
    with pytest.raises(MTError):
        mp.logpost_grad(torch.zeros((mp.max_chains + 1, mp.P), device=DEV))


def test_ragged_rays_small_grid_and_zero_counts(problems):
    """n = 3 grid, 1000 rays (not a multiple of the block), zero counts,
    detectors near the walls, a vertical ray, axis-parallel rays."""
    base = problems("tiny")
    X = inputs.quantize([0.0, 40.0, 100.0]).astype(np.float32)
    rng = np.random.default_rng(11)
    dets = inputs.quantize(np.array([[0.5, 0.5], [99.25, 50.0], [40.0, 40.0], [70.0, 3.0]]))
    dets = np.concatenate([dets, np.zeros((4, 1))], 1).astype(np.float32)
    R = 1000
    th = rng.uniform(0, 1.3, R)
    ph = rng.uniform(0, 2 * np.pi, R)
    d = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], 1)
    d[0] = [0, 0, 1]
    d[1] = [np.sin(0.5), 0, np.cos(0.5)]
    d[2] = [0, -np.sin(0.7), np.cos(0.7)]
    prob = dict(base, node_x=X, node_y=X.copy(), det_xyz=dets, ray_det=rng.integers(0, 4, R).astype(np.int32),
                ray_dir=d.astype(np.float32), ray_w=rng.uniform(200, 2000, R).astype(np.float32),
                counts=np.where(rng.random(R) < 0.2, 0, rng.integers(1, 900, R)).astype(np.int32))
    op = oracle.Problem(prob)
    mp = Problem(prob, device=0, max_chains=3)
    xx, yy = np.meshgrid(X.astype(np.float64), X.astype(np.float64), indexing="ij")
    H = np.stack([np.stack([110 + 0.2 * xx - 0.1 * yy + 3 * c, 160 + 0.1 * yy + 5 * np.sin(xx / 20) + c])
                  for c in range(3)]).astype(np.float32)
    L_d, _ = mp.path_lengths(torch.from_numpy(H).to(DEV))
    L_o, _ = op.path_lengths(H.astype(np.float64))
    assert np.all(np.abs(L_d.cpu().numpy() - L_o).max(2) <= 1e-5 * L_o.sum(2))
    ll_d, G_d = mp.loglik_heights(torch.from_numpy(H).to(DEV))
    out = op.loglik_grad_H(H.astype(np.float64))
    assert np.allclose(ll_d.cpu().numpy(), out["ll_dev"], rtol=1e-4)
    for c in range(3):
        assert rel_l2(G_d.cpu().numpy()[c].astype(np.float64), out["dldH"][c]) <= 1e-3
    for q in range(0, R, 37):
        assert np.array_equal(mp.debug_traversal(q)[0], op.traversal(q)[0])


def test_nonfinite_state_sets_status_only_for_that_chain(gpu):
    mp = gpu("small", max_chains=64)
    cfg = inputs.CONFIGS["small"]
    from paper_2603_28907_b200 import inputs as I
    x = torch.from_numpy(I.chain_states(mp_x_true(), 4, cfg.seed)).to(DEV)
    x[2, 5] = float("nan")
    status = torch.zeros(4, dtype=torch.int32, device=DEV)
    lp, g = mp.logpost_grad(x, status=status)
    st = status.cpu().numpy()
    assert st[2] & 1 and st[0] == 0 and st[1] == 0 and st[3] == 0
    assert np.isfinite(lp.cpu().numpy()[[0, 1, 3]]).all()


def mp_x_true():
    return inputs.make_problem("small")["x_true"]


def test_ray_shards_sum_to_whole(gpu, problems):
    prob = problems("small")
    R = len(prob["ray_det"])
    cfg = inputs.CONFIGS["small"]
    whole = gpu("small", max_chains=8)
    parts = [Problem(prob, device=0, max_chains=8, ray_lo=lo, ray_hi=hi)
             for lo, hi in ((0, 5000), (5000, 11111), (11111, R))]
    x = torch.from_numpy(inputs.chain_states(prob["x_true"], 8, cfg.seed)).to(DEV)
    lp, g = whole.logpost_grad(x)
    lps, gs = zip(*[p.logpost_grad(x) for p in parts])
    assert np.allclose(sum(l.cpu().numpy() for l in lps), lp.cpu().numpy(), rtol=1e-6)
    gsum = sum(v.cpu().numpy().astype(np.float64) for v in gs)
    for c in range(8):
        assert rel_l2(gsum[c], g.cpu().numpy()[c].astype(np.float64)) < 1e-5


# ---------------------------------------------------------------------------
# a9 statistics kernels against plain numpy
# ---------------------------------------------------------------------------
def test_stats_kernels_match_numpy(gpu):
    mp = gpu("small", max_chains=64)
    C, P = 64, mp.P
    rng = np.random.default_rng(4)
    draws = rng.standard_normal((12, C, P)).astype(np.float32)
    acc = rng.uniform(0, 1, (12, C)).astype(np.float32)
    mean = torch.zeros((C, P), device=DEV)
    m2 = torch.zeros((C, P), device=DEV)
    accf = torch.zeros(2, dtype=torch.int64, device=DEV)
    for it in range(12):
        mp.stats_update(C, x=torch.from_numpy(draws[it]).to(DEV), accept_prob=torch.from_numpy(acc[it]).to(DEV),
                        n_prev=it, mean=mean, m2=m2, acc_fixed=accf)
    torch.cuda.synchronize()
    assert np.allclose(mean.cpu().numpy(), draws.mean(0), atol=1e-5)
    assert np.allclose(m2.cpu().numpy() / 11, draws.var(0, ddof=1), rtol=1e-4, atol=1e-5)
    s, n = accf.cpu().tolist()
    ref = int(np.sum(np.rint(acc.astype(np.float64) * 4294967296.0).astype(np.int64)))
    assert s == ref and n == 12 * C            # exact integer sums
    part = mp.rhat_partials(C, mean, m2, 12).cpu().numpy()
    cm = draws.astype(np.float64).mean(0)
    assert np.allclose(part[0], cm.sum(0), rtol=1e-5, atol=1e-4)
    assert np.allclose(part[1], (cm ** 2).sum(0), rtol=1e-5, atol=1e-4)
    assert np.allclose(part[2], draws.astype(np.float64).var(0, ddof=1).sum(0), rtol=1e-4)


def test_hmc_driver_runs_and_adapts(gpu, problems):
    """ChainShard: dual-averaging warm-up then sampling on Small; acceptance
    near the 0.8 target, finite R-hat, chains stay finite."""
    from paper_2603_28907_b200.hmc import ChainShard
    prob = problems("small")
    cfg = inputs.CONFIGS["small"]
    mp = gpu("small", max_chains=64)
    x0 = inputs.chain_states(prob["x_true"], 64, cfg.seed, super_size=8)
    sh = ChainShard(mp, x0, seed=inputs.philox_key(cfg), L=10, eps0=cfg.eps)
    out = sh.run(60, 20)
    assert 0.55 < np.mean(out["warmup_accept"][-10:]) < 0.95
    assert np.all(np.isfinite(out["rhat"])) and out["rhat"].min() > 0.9
    assert torch.isfinite(sh.x).all() and torch.isfinite(sh.logp).all()


# ---------------------------------------------------------------------------
# ray sharding with the in-library NCCL communicator (one GPU: a one-rank
# communicator runs the all-reduce code path; multi-rank logic: test_dist_cpu)
# ---------------------------------------------------------------------------
def test_one_rank_communicator_reproduces_unsharded_hmc(gpu, problems):
    from paper_2603_28907_b200 import comm_unique_id
    from paper_2603_28907_b200.hmc import ray_sharded_problem
    name, C = "small", 8
    prob = problems(name)
    cfg = inputs.CONFIGS[name]
    plain = Problem(prob, device=0, max_chains=C)
    shard = ray_sharded_problem(prob, 0, 1, 0, C)       # world 1: no communicator
    shard.attach_comm(comm_unique_id(), 0, 1)             # ... attach one explicitly
    x0 = torch.from_numpy(inputs.chain_states(prob["x_true"], C, cfg.seed)).to(DEV)
    out = []
    for pb in (plain, shard):
        x = x0.clone()
        logp, grad = pb.logpost_grad(x)
        eps = torch.full((C,), sampling_eps(name), dtype=torch.float32, device=DEV)
        ap, acc = pb.hmc_step(x, logp, grad, eps, 10, inputs.philox_key(cfg), 5)
        torch.cuda.synchronize()
        out.append((x.cpu().numpy(), logp.cpu().numpy(), grad.cpu().numpy(), ap.cpu().numpy()))
    # (not bit-identical: the adjoint's float atomics sum in run-dependent order)
    (x1, lp1, g1, a1), (x2, lp2, g2, a2) = out
    for c in range(C):
        assert rel_l2(x2[c].astype(np.float64), x1[c].astype(np.float64)) < 1e-5
        assert rel_l2(g2[c].astype(np.float64), g1[c].astype(np.float64)) < 1e-4
    assert np.allclose(lp2, lp1, rtol=2e-6)      # (atomic-order rounding only; logp tolerance is 1e-4)
    assert np.allclose(a2, a1, atol=1e-3)
    shard.detach_comm()


def test_ray_shards_partition_and_sum_ray_sharded_config(gpu, problems):
    """configs[4] split as for 4 GPUs (hmc.ray_shards): the shards' partial
    log-posteriors and gradients (prior on shard 0 only) sum to the whole."""
    from paper_2603_28907_b200.hmc import ray_shards
    prob = problems("ray_sharded")
    R = len(prob["ray_det"])
    sh = ray_shards(R, 4)
    assert sh[0][0] == 0 and sh[-1][1] == R and all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
    whole = gpu("ray_sharded")
    x = torch.from_numpy(inputs.chain_states(prob["x_true"], 1, inputs.CONFIGS["ray_sharded"].seed)).to(DEV)
    lp, g = whole.logpost_grad(x)
    lps, gs = [], []
    for lo, hi in sh:
        part = Problem(prob, device=0, max_chains=1, ray_lo=lo, ray_hi=hi)
        a, b = part.logpost_grad(x)
        lps.append(a.cpu().numpy())
        gs.append(b.cpu().numpy().astype(np.float64))
        del part
    assert np.allclose(sum(lps), lp.cpu().numpy(), rtol=1e-7)
    assert rel_l2(sum(gs)[0], g.cpu().numpy()[0].astype(np.float64)) < 1e-5


# ---------------------------------------------------------------------------
# hierarchical r_l: state (x_0, x_1, ρ_0, ρ_1)
# ---------------------------------------------------------------------------
def sampled_r_states(prob, C, seed, rho=(2.5, 2.0)):
    x = inputs.chain_states(prob["x_true"], C, seed)
    rng = np.random.default_rng(seed + 99)
    r = np.asarray(rho)[None] + 0.3 * rng.standard_normal((C, 2))
    return np.concatenate([x, r.astype(np.float32)], axis=1).astype(np.float32)


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_sampled_r_logpost_grad(gpu, oracle_problem, problems, name):
    op = oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    mp = Problem(problems(name), device=0, max_chains=cfg.chains, sample_r=True)
    assert mp.P == op.P + 2
    v = sampled_r_states(op.prob, cfg.chains, cfg.seed)
    logp, grad = mp.logpost_grad(torch.from_numpy(v).to(DEV))
    ref = op.logpost_grad_r(v.astype(np.float64))
    lp, g = logp.cpu().numpy(), grad.cpu().numpy().astype(np.float64)
    for c in range(cfg.chains):
        assert abs(lp[c] - ref["logp"][c]) <= 1e-4 * abs(ref["logp"][c]), (c, lp[c], ref["logp"][c])
        assert rel_l2(g[c], ref["grad"][c]) <= 1e-3, (c, rel_l2(g[c], ref["grad"][c]))
        # the two hyper-parameter components on their own (relative to the chain's gradient scale)
        assert np.abs(g[c, -2:] - ref["grad"][c, -2:]).max() <= 1e-3 * np.abs(ref["grad"][c]).max()


def test_sampled_r_leapfrog_10_steps(gpu, oracle_problem, problems):
    name, C = "small", 8
    op = oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    mp = Problem(problems(name), device=0, max_chains=C, sample_r=True)
    v0 = sampled_r_states(op.prob, C, cfg.seed)
    x = torch.from_numpy(v0).to(DEV)
    p = mp.draw_momenta(C, inputs.philox_key(cfg), 0)
    p0 = p.cpu().numpy().astype(np.float64)
    logp, grad = mp.logpost_grad(x)
    e = sampling_eps(name)
    eps = torch.full((C,), e, dtype=torch.float32, device=DEV)
    mp.leapfrog(x, p, logp, grad, eps, 10)
    lg = lambda vv: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad_r(vv))  # noqa: E731
    xo, po, lpo, go = oracle.leapfrog(v0.astype(np.float64), p0, e, 10, lg)
    xd = x.cpu().numpy().astype(np.float64)
    for c in range(C):
        assert rel_l2(xd[c], xo[c]) <= 1e-3, (c, rel_l2(xd[c], xo[c]))
    ref = op.logpost_grad_r(xd)
    assert np.allclose(logp.cpu().numpy(), ref["logp"], rtol=1e-4)
    for c in range(C):
        assert rel_l2(grad.cpu().numpy()[c].astype(np.float64), ref["grad"][c]) <= 1e-3


def test_sampled_r_hmc_step_with_and_without_communicator(gpu, oracle_problem, problems):
    """mt_hmc_step with sampled r: the fused path (k_finish_r) and the ray-shard
    path (k_kick_r after a one-rank NCCL all-reduce) agree; the trajectory's end
    state matches the oracle's log-posterior/gradient at that state."""
    from paper_2603_28907_b200 import comm_unique_id
    name, C = "small", 8
    op = oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    prob = problems(name)
    plain = Problem(prob, device=0, max_chains=C, sample_r=True)
    shard = Problem(prob, device=0, max_chains=C, sample_r=True)
    shard.attach_comm(comm_unique_id(), 0, 1)
    v0 = torch.from_numpy(sampled_r_states(op.prob, C, cfg.seed)).to(DEV)
    out = []
    for pb in (plain, shard):
        x = v0.clone()
        logp, grad = pb.logpost_grad(x)
        eps = torch.full((C,), sampling_eps(name), dtype=torch.float32, device=DEV)
        ap, acc = pb.hmc_step(x, logp, grad, eps, 10, inputs.philox_key(cfg), 7)
        torch.cuda.synchronize()
        out.append((x.cpu().numpy().astype(np.float64), logp.cpu().numpy(), ap.cpu().numpy()))
    shard.detach_comm()
    (x1, lp1, a1), (x2, lp2, a2) = out
    for c in range(C):
        assert rel_l2(x2[c], x1[c]) < 1e-5
    assert np.allclose(lp2, lp1, rtol=2e-6)      # (atomic-order rounding only; logp tolerance is 1e-4)
    assert np.all((a1 >= 0) & (a1 <= 1)) and np.allclose(a1, a2, atol=1e-3)
    ref = op.logpost_grad_r(x1)
    assert np.allclose(lp1, ref["logp"], rtol=1e-4)


# ---------------------------------------------------------------------------
# batched NUTS against the oracle's one-chain NUTS
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,C,max_depth", [("tiny", 4, 5), ("small", 16, 4)])
def test_nuts_step_matches_oracle(gpu, oracle_problem, name, C, max_depth):
    """Kernel NUTS vs the oracle's NUTS from the same state with the same Philox
    streams.  Long trajectories amplify the fp32/fp64 evaluation differences
    exponentially (tools/nuts_debug.py: |Δθ| grows 1e-6 -> 1e-3 over ~20 leaves at
    2x the tuned ε and then flips a multinomial choice), so trees are kept to
    2^max_depth <= 32 leaves at the tuned ε; chains whose tree decisions agree must
    land on the same state."""
    mp, op = gpu(name), oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    x0 = inputs.chain_states(op.prob["x_true"], C, cfg.seed)
    seed, it = inputs.philox_key(cfg), 11
    e = sampling_eps(name)
    x = torch.from_numpy(x0).to(DEV)
    logp, grad = mp.logpost_grad(x)
    eps = torch.full((C,), e, dtype=torch.float32, device=DEV)
    acc, depth, nl = mp.nuts_step(x, logp, grad, eps, max_depth, seed, it)
    torch.cuda.synchronize()
    xd, depth, nl, acc = x.cpu().numpy().astype(np.float64), depth.cpu().numpy(), nl.cpu().numpy(), acc.cpu().numpy()
    lg1 = lambda th: (lambda o: (o["logp"][0], o["grad"][0]))(op.logpost_grad(th[None]))  # noqa: E731
    agree = 0
    for c in range(C):
        lp0, g0 = lg1(x0[c].astype(np.float64))
        ref = oracle.nuts_step(x0[c], lp0, g0, e, lg1, seed, it, c, max_depth=max_depth)
        if ref["depth"] == depth[c] and ref["n_leaves"] == nl[c]:
            agree += 1
            assert rel_l2(xd[c], ref["x"]) <= 1e-3, (c, rel_l2(xd[c], ref["x"]))
            assert acc[c] == pytest.approx(ref["accept_stat"], abs=2e-3)
    # the tree decisions compare fp32 against fp64 quantities: allow the rare
    # chain whose U-turn or selection sits on a threshold to differ
    assert agree >= max(C - 1, int(0.75 * C)), (agree, C)
    ref_lp = op.logpost_grad(xd)
    assert np.allclose(logp.cpu().numpy(), ref_lp["logp"], rtol=1e-4)   # returned logp is that of x


def test_nuts_driver_runs_and_adapts(gpu, problems):
    """ChainShard(sampler="nuts") on Small: dual averaging on the NUTS acceptance
    statistic reaches the 0.8 target neighbourhood, trees stay under the cap,
    chains stay finite."""
    from paper_2603_28907_b200.hmc import ChainShard
    prob = problems("small")
    cfg = inputs.CONFIGS["small"]
    mp = gpu("small", max_chains=64)
    x0 = inputs.chain_states(prob["x_true"], 64, cfg.seed, super_size=8)
    sh = ChainShard(mp, x0, seed=inputs.philox_key(cfg), L=10, eps0=sampling_eps("small"), sampler="nuts",
                    max_depth=5)
    out = sh.run(30, 5)
    assert 0.5 < np.mean(out["warmup_accept"][-10:]) < 0.98
    d = sh.depth.cpu().numpy()
    assert d.min() >= 1 and d.max() <= 5
    assert torch.isfinite(sh.x).all() and torch.isfinite(sh.logp).all()


def test_chain_shards_reproduce_the_unsharded_hmc_step(gpu, problems):
    """Chain sharding (configs[3], §9): a rank's chains are a contiguous slice with
    chain_offset = its first global id; Philox streams depend on the global id only,
    so two 32-chain shards reproduce one 64-chain HMC step (up to the summation
    order of the float atomics)."""
    prob = problems("small")
    cfg = inputs.CONFIGS["small"]
    mp = gpu("small")
    x0 = torch.from_numpy(inputs.chain_states(prob["x_true"], 64, cfg.seed)).to(DEV)
    eps = torch.full((64,), sampling_eps("small"), dtype=torch.float32, device=DEV)
    seed = inputs.philox_key(cfg)
    xa = x0.clone()
    lpa, ga = mp.logpost_grad(xa)
    apa, acca = mp.hmc_step(xa, lpa, ga, eps, 10, seed, 3)
    xb = x0.clone()
    lpb, gb = mp.logpost_grad(xb)
    aps, accs = [], []
    for lo in (0, 32):
        ap, acc = mp.hmc_step(xb[lo:lo + 32], lpb[lo:lo + 32], gb[lo:lo + 32], eps[lo:lo + 32], 10, seed, 3,
                              chain_offset=lo)
        aps.append(ap)
        accs.append(acc)
    apb, accb = torch.cat(aps), torch.cat(accs)
    assert torch.allclose(apa, apb, rtol=0, atol=1e-3)
    close = (apa - apb).abs() < 1e-4
    assert torch.equal(acca[close], accb[close])
    assert float((xa - xb).norm() / xa.norm()) < 1e-6


@pytest.mark.parametrize("mode", ["plain", "one_rank_comm", "few_chains"])
def test_cuda_graph_capture_and_replay(gpu, problems, mode):
    """The evaluation and leapfrog entry points are stream-ordered with no host
    synchronisation, so they can be captured into a CUDA graph (with the
    in-library NCCL all-reduce when a communicator is attached) and replayed:
    a replayed 10-step leapfrog equals the eager one."""
    from paper_2603_28907_b200 import comm_unique_id
    prob = problems("small")
    cfg = inputs.CONFIGS["small"]
    C = 4 if mode == "few_chains" else 32
    pb = Problem(prob, device=0, max_chains=C)
    if mode == "one_rank_comm":
        pb.attach_comm(comm_unique_id(), 0, 1)
    x0 = torch.from_numpy(inputs.chain_states(prob["x_true"], C, cfg.seed)).to(DEV)
    p0 = torch.from_numpy(np.random.default_rng(3).standard_normal((C, pb.P)).astype(np.float32)).to(DEV)
    eps = torch.full((C,), sampling_eps("small"), dtype=torch.float32, device=DEV)
    # eager reference
    xe, pe = x0.clone(), p0.clone()
    lpe, ge = pb.logpost_grad(xe)
    pb.leapfrog(xe, pe, lpe, ge, eps, 10)
    # static buffers, warm-up on a side stream, capture, replay
    xs, ps = x0.clone(), p0.clone()
    lps = torch.empty(C, dtype=torch.float64, device=DEV)
    gs = torch.empty_like(xs)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        pb.logpost_grad(xs, lps, gs)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):      # (the binding launches on the current = capture stream)
        pb.logpost_grad(xs, lps, gs)
        pb.leapfrog(xs, ps, lps, gs, eps, 10)
    xs.copy_(x0)
    ps.copy_(p0)
    graph.replay()
    torch.cuda.synchronize()
    assert float((xs - xe).norm() / xe.norm()) < 1e-5
    assert np.allclose(lps.cpu().numpy(), lpe.cpu().numpy(), rtol=1e-6)
    if mode == "one_rank_comm":
        pb.detach_comm()


def test_gpu_properties_on_random_geometries(gpu, oracle_problem):
    """Property tests on the device path: for random (rough) ordered
    surfaces, every ray's muck / air / rock lengths are non-negative and sum to
    its in-box length, and they equal the oracle's within the north_star bound."""
    from hypothesis import HealthCheck, given, settings
    from hypothesis import strategies as st
    from test_oracle_properties import random_heights
    mp, op = gpu("small"), oracle_problem("small")
    s_exit = np.array([op.ray_extent(q)[0] for q in range(op.R)])

    @settings(max_examples=8, deadline=None, derandomize=True,
              suppress_health_check=[HealthCheck.function_scoped_fixture])
    @given(seed=st.integers(0, 2 ** 31 - 1), rough=st.floats(0.0, 1.0))
    def check(seed, rough):
        H = random_heights(np.random.default_rng(seed), op.nx, rough=rough).astype(np.float32)
        L, O = mp.path_lengths(torch.from_numpy(H[None]).to(DEV))
        L = L.cpu().numpy()[0].astype(np.float64)
        assert np.all(L >= -1e-3)
        assert np.allclose(L.sum(1), s_exit, rtol=1e-5, atol=1e-3)
        Lo, _ = op.path_lengths(H[None].astype(np.float64))
        assert np.max(np.abs(L - Lo[0]) / s_exit[:, None]) <= 1e-5
    check()
