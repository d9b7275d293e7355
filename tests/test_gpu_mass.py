"""GPU parity of the diagonal inverse mass (R19b; NumPyro's adapted diagonal
mass for the paper's sampler) in every momentum-carrying kernel:
Philox momenta p = z / sqrt(m), fused and unfused leapfrog (fixed r, sampled
r, non-centred, few chains), HMC and NUTS, against the oracle with the same
inverse mass; and the warm-up window adaptation of ChainShard."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs  # noqa: E402

DEV = "cuda:0"


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def minv_for(P, seed=0):
    return np.random.default_rng(seed).uniform(0.3, 3.0, P).astype(np.float32)


def test_momenta_with_mass(problems):
    prob = problems("small")
    mp = Problem(prob, device=0, max_chains=8)
    m = minv_for(mp.P)
    mp.set_inverse_mass(torch.from_numpy(m).to(DEV))
    p = mp.draw_momenta(8, 99, 3).cpu().numpy().astype(np.float64)
    for c in range(8):
        ref = oracle.momenta(mp.P, 99, 3, c) / np.sqrt(m.astype(np.float64))
        assert np.allclose(p[c], ref, rtol=1e-6, atol=1e-6)
    mp.set_inverse_mass(None)
    p2 = mp.draw_momenta(8, 99, 3).cpu().numpy().astype(np.float64)
    assert np.allclose(p2[0], oracle.momenta(mp.P, 99, 3, 0), atol=1e-6)


@pytest.mark.parametrize("name,C,mode", [("tiny", 4, "fixed"), ("small", 16, "fixed"), ("small", 16, "sample_r"),
                                         ("small", 4, "noncentred")])
def test_hmc_step_with_mass_matches_oracle(problems, oracle_problem, name, C, mode):
    """C = 4 exercises the few-chain multi-block kernels, 16 the fused ones; the
    ρ momenta of sampled r and the non-centred kick take the mass too."""
    prob = problems(name)
    op = oracle_problem(name)
    cfg = inputs.CONFIGS[name]
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
    if mode == "sample_r":
        x0 = np.concatenate([x0, np.tile([[2.5, 2.0]], (C, 1))], axis=1).astype(np.float32)
        lg = lambda v: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad_r(v))  # noqa: E731
        mp = Problem(prob, device=0, max_chains=C, sample_r=True)
    elif mode == "noncentred":
        from paper_2603_28907_b200.hmc import noncentred_state
        x0 = noncentred_state(x0, (2.5, 2.0), cfg.n, cfg.n)
        lg = lambda v: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad_ncp(v))  # noqa: E731
        mp = Problem(prob, device=0, max_chains=C, noncentred=True)
    else:
        lg = lambda v: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad(v))  # noqa: E731
        mp = Problem(prob, device=0, max_chains=C)
    m = minv_for(mp.P, 1)
    mp.set_inverse_mass(torch.from_numpy(m).to(DEV))
    e = 1e-4 if mode == "noncentred" else 5e-6
    seed, it = inputs.philox_key(cfg), 4
    x = torch.from_numpy(x0.copy()).to(DEV)
    lp, g = mp.logpost_grad(x)
    eps = torch.full((C,), e, dtype=torch.float32, device=DEV)
    ap, acc = mp.hmc_step(x, lp, g, eps, 10, seed, it)
    xr, apr, accr, lpr, dH = oracle.hmc_step(x0.astype(np.float64), e, 10, lg, seed, it, minv=m)
    xd, apd, accd = x.cpu().numpy().astype(np.float64), ap.cpu().numpy(), acc.cpu().numpy().astype(bool)
    for c in range(C):
        if abs(np.log(oracle.mh_uniform(seed, it, c)) + dH[c]) > 0.05:   # decision away from the threshold
            assert accd[c] == accr[c], c
            assert rel_l2(xd[c], xr[c]) <= 1e-3, (c, rel_l2(xd[c], xr[c]))
        assert abs(apd[c] - apr[c]) <= 2e-3 + 2e-2 * apr[c], (c, apd[c], apr[c])


def test_nuts_with_mass_matches_oracle(problems, oracle_problem):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    cfg = inputs.CONFIGS["tiny"]
    C, max_depth, e, seed, it = 4, 4, 2e-3, inputs.philox_key(cfg), 7
    mp = Problem(prob, device=0, max_chains=C)
    m = minv_for(mp.P, 2)
    mp.set_inverse_mass(torch.from_numpy(m).to(DEV))
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
    x = torch.from_numpy(x0).to(DEV)
    lp, g = mp.logpost_grad(x)
    acc, depth, nl = mp.nuts_step(x, lp, g, torch.full((C,), e, dtype=torch.float32, device=DEV), max_depth,
                                  seed, it)
    xd = x.cpu().numpy().astype(np.float64)
    lg1 = lambda th: (lambda o: (o["logp"][0], o["grad"][0]))(op.logpost_grad(th[None]))  # noqa: E731
    agree = 0
    for c in range(C):
        lp0, g0 = lg1(x0[c].astype(np.float64))
        ref = oracle.nuts_step(x0[c], lp0, g0, e, lg1, seed, it, c, max_depth=max_depth, minv=m)
        if ref["depth"] == depth[c].item() and ref["n_leaves"] == nl[c].item():
            agree += 1
            assert rel_l2(xd[c], ref["x"]) <= 1e-3
            assert acc[c].item() == pytest.approx(ref["accept_stat"], abs=2e-3)
    assert agree >= C - 1, agree


def test_chainshard_adapts_a_diagonal_mass(problems):
    """Warm-up windows estimate M^-1 from pooled within-chain variances: the
    muck-top latents (∂H0/∂x0 ≈ 10× ∂H1/∂x1) get a smaller
    posterior variance than the cave-back latents; sampling then stays finite."""
    from paper_2603_28907_b200.hmc import ChainShard
    prob = problems("small")
    cfg = inputs.CONFIGS["small"]
    mp = Problem(prob, device=0, max_chains=64)
    x0 = inputs.chain_states(prob["x_true"], 64, cfg.seed, super_size=8)
    sh = ChainShard(mp, x0, seed=inputs.philox_key(cfg), L=10, eps0=cfg.eps, adapt_mass=True)
    out = sh.run(150, 20)
    m = sh.minv.cpu().numpy()
    N = mp.P // 2
    assert np.all(m > 0) and np.all(np.isfinite(m))
    assert np.median(m[:N]) < np.median(m[N:])
    assert np.isfinite(out["eps"]) and out["eps"] > 0
    assert torch.isfinite(sh.x).all() and torch.isfinite(sh.logp).all()
    assert 0.4 < np.mean(out["warmup_accept"][-10:]) < 0.99


def test_leapfrog_with_extreme_mass(problems, oracle_problem):
    """Inverse masses spanning six decades (1e-3 .. 1e3) in the fused leapfrog."""
    prob = problems("small")
    op = oracle_problem("small")
    C = 16
    mp = Problem(prob, device=0, max_chains=C)
    m = np.exp(np.random.default_rng(4).uniform(np.log(1e-3), np.log(1e3), mp.P)).astype(np.float32)
    mp.set_inverse_mass(torch.from_numpy(m).to(DEV))
    x0 = inputs.chain_states(prob["x_true"], C, inputs.CONFIGS["small"].seed)
    p0 = np.random.default_rng(5).standard_normal(x0.shape).astype(np.float32)
    e = 2e-7
    x = torch.from_numpy(x0.copy()).to(DEV)
    p = torch.from_numpy(p0.copy()).to(DEV)
    lp, g = mp.logpost_grad(x)
    mp.leapfrog(x, p, lp, g, torch.full((C,), e, dtype=torch.float32, device=DEV), 10)
    lg = lambda v: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad(v))  # noqa: E731
    xo, po, lpo, _ = oracle.leapfrog(x0.astype(np.float64), p0.astype(np.float64), e, 10, lg, minv=m)
    xd = x.cpu().numpy().astype(np.float64)
    for c in range(C):
        assert rel_l2(xd[c], xo[c]) <= 1e-3, (c, rel_l2(xd[c], xo[c]))
        assert np.linalg.norm(xd[c] - xo[c]) / np.linalg.norm(xo[c] - x0[c]) < 0.05
