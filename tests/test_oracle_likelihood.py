"""Oracle pins: Poisson likelihood, log-posterior and the
reverse-mode gradient, against scipy's Poisson log-pmf and central finite
differences of the oracle's own forward value.
"""
import numpy as np
import pytest
from scipy.special import gammaln
from scipy.stats import poisson

import oracle
from paper_2603_28907_b200 import inputs


def test_poisson_spot_value():
    # S:390 prints -1.90278 for log Poisson(2; 3); the correct value is 2 ln 3 - 3 - ln 2
    assert poisson.logpmf(2, 3.0) == pytest.approx(2 * np.log(3) - 3 - np.log(2), rel=1e-14)
    assert poisson.logpmf(2, 3.0) == pytest.approx(-1.4959226, abs=1e-7)


def test_loglik_matches_scipy(problems):
    base = dict(problems("small"))
    rng = np.random.default_rng(2)
    counts = base["counts"].copy()
    counts[rng.choice(len(counts), 50, replace=False)] = 0          # C = 0 rays
    base["counts"] = counts
    op = oracle.Problem(base)
    H = inputs.perturbed_heights(base["H_true"], 3, 8, scale=2.0).astype(np.float64)
    _, O = op.path_lengths(H)
    out = op.loglik_grad_H(H)
    lam = base["ray_w"].astype(np.float64)[None] * np.exp(-O / base["att_len"])
    ref = poisson.logpmf(counts[None], lam).sum(1)
    assert np.allclose(out["ll_std"], ref, rtol=1e-12)
    c = counts.astype(np.float64)
    off = np.sum(np.where(c > 0, c * np.log(np.maximum(c, 1)), 0) - c - gammaln(c + 1))
    assert np.allclose(out["ll_dev"], ref - off, rtol=1e-10, atol=1e-6)
    assert op.loglik_offset() == pytest.approx(off, rel=1e-12)
    assert np.all(out["ll_dev"] <= 0)


def well_conditioned(op, H, h):
    """Nodes whose FD step moves no crossing near a cell edge / grazing."""
    _, _, mg = op.path_lengths(H, with_min_g1=True)
    return np.nanmin(mg) > 1e-3


def test_gradient_H_vs_fd(problems):
    base = problems("tiny")
    op = oracle.Problem(base)
    H = inputs.perturbed_heights(base["H_true"], 1, 21, scale=2.0).astype(np.float64)
    assert well_conditioned(op, H, 1e-4)
    g = op.loglik_grad_H(H)["dldH"][0]
    h = 1e-4
    errs = []
    for l in (0, 1):
        for i in range(op.nx):
            for j in range(op.ny):
                Hp = H.copy()
                Hm = H.copy()
                Hp[0, l, i, j] += h
                Hm[0, l, i, j] -= h
                fd = (op.loglik_grad_H(Hp)["ll_dev"][0] - op.loglik_grad_H(Hm)["ll_dev"][0]) / (2 * h)
                errs.append(abs(fd - g[l, i, j]) / (abs(g).max()))
    assert max(errs) < 1e-6


def test_gradient_x_vs_fd(problems):
    base = problems("tiny")
    op = oracle.Problem(base)
    x = inputs.chain_states(base["x_true"], 2, 1, scale=0.05).astype(np.float64)
    out = op.logpost_grad(x)
    h = 1e-6
    rng = np.random.default_rng(0)
    for c in range(2):
        for k in rng.choice(op.P, 40, replace=False):
            xp = x.copy()
            xm = x.copy()
            xp[c, k] += h
            xm[c, k] -= h
            fd = (op.logpost_grad(xp)["logp"][c] - op.logpost_grad(xm)["logp"][c]) / (2 * h)
            assert fd == pytest.approx(out["grad"][c, k], rel=1e-5, abs=1e-5 * np.abs(out["grad"][c]).max())


def test_logpost_is_loglik_plus_prior(problems):
    base = problems("small")
    op = oracle.Problem(base)
    x = inputs.chain_states(base["x_true"], 3, 2).astype(np.float64)
    out = op.logpost_grad(x)
    H = np.stack([op.heights(xc)[0] for xc in x])
    ll = op.loglik_grad_H(H)["ll_dev"]
    pr = np.array([sum(oracle.prior_surface(xc.reshape(2, op.nx, op.ny)[l], op.car_r[l])[0]
                       for l in (0, 1)) for xc in x])
    assert np.allclose(out["logp"], ll + pr, rtol=1e-13)
    assert np.allclose(out["ll_std"] - out["ll_dev"], op.loglik_offset(), rtol=1e-10)
