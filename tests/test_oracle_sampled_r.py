"""Oracle pins for the hierarchical CAR dependence r_l (SURVEY
§8(f) f2; readings R13b/R13c in DESIGN.md): r_l = logistic(ρ_l) with
r_l ~ Unif(0,1), x_l | r_l ~ N(0, Q(r_l)^-1), heights through σ(r_l).

Pinned against: dense matrix identities for the r-derivatives of the torus
spectrum (d ln det Q/dr = -tr(Q⁻¹A), dΣ_ii/dr = (Q⁻¹AQ⁻¹)_ii with numpy inv),
the already-pinned fixed-r oracle (same r ⇒ same value up to the hyperprior
term and same x-gradient), scipy's logistic pdf for the ρ hyperprior, and
central finite differences of the full log-posterior in x and ρ.
"""
import numpy as np
import pytest
from scipy.stats import logistic

import oracle
from paper_2603_28907_b200 import inputs
from test_oracle_prior import dense_Q, torus_adjacency


@pytest.mark.parametrize("nr,nc,r", [(3, 3, 0.3), (4, 4, 0.8), (4, 6, 0.95), (8, 8, 0.5)])
def test_spectrum_derivatives_vs_dense(nr, nc, r):
    A = torus_adjacency(nr, nc)
    Qi = np.linalg.inv(dense_Q(nr, nc, r))
    s, ds, ld, dld = oracle.torus_spectrum_dr(nr, nc, r)
    assert s ** 2 == pytest.approx(Qi[0, 0], rel=1e-12)
    assert ld == pytest.approx(np.linalg.slogdet(dense_Q(nr, nc, r))[1], rel=1e-12)
    assert dld == pytest.approx(-np.trace(Qi @ A), rel=1e-11)                 # d ln det Q = tr(Q⁻¹ dQ)
    dSii = (Qi @ A @ Qi)[0, 0]                                              # dQ⁻¹/dr = Q⁻¹ A Q⁻¹
    assert 2 * s * ds == pytest.approx(dSii, rel=1e-11)


def _v(x, rho):
    return np.concatenate([x, np.broadcast_to(rho, (x.shape[0], 2))], axis=1)


def test_sampled_r_reduces_to_fixed_r(problems):
    base = problems("tiny")
    op = oracle.Problem(base)
    x = inputs.chain_states(base["x_true"], 2, 1, scale=0.05).astype(np.float64)
    r = op.car_r[0]
    assert op.car_r[1] == r
    rho = np.log(r / (1 - r))
    fixed = op.logpost_grad(x)
    samp = op.logpost_grad_r(_v(x, rho))
    hyper = 2 * logistic.logpdf(rho)            # ln r(1-r) = logistic density of ρ, per surface
    assert np.allclose(samp["logp"], fixed["logp"] + hyper, rtol=1e-12)
    assert np.allclose(samp["grad"][:, :op.P], fixed["grad"], rtol=1e-10, atol=1e-9)


def test_sampled_r_gradient_vs_fd(problems):
    base = problems("tiny")
    op = oracle.Problem(base)
    x = inputs.chain_states(base["x_true"], 2, 1, scale=0.05).astype(np.float64)
    v = _v(x, np.array([1.5, 2.5]))
    out = op.logpost_grad_r(v)
    rng = np.random.default_rng(3)
    ks = list(rng.choice(op.P, 20, replace=False)) + [op.P, op.P + 1]
    for c in range(2):
        for k in ks:
            h = 1e-6 if k < op.P else 1e-5
            vp, vm = v.copy(), v.copy()
            vp[c, k] += h
            vm[c, k] -= h
            fd = (op.logpost_grad_r(vp)["logp"][c] - op.logpost_grad_r(vm)["logp"][c]) / (2 * h)
            assert fd == pytest.approx(out["grad"][c, k], rel=1e-5, abs=1e-5 * np.abs(out["grad"][c]).max()), k
