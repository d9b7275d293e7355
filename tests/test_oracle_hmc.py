"""Oracle pins: leapfrog integrator, HMC transition and Philox4x32-10.

Leapfrog on a Gaussian target has a closed-form linear map; reversibility and
O(ε²) energy error are textbook invariants; HMC moments on N(0, I) are
statistical; Philox is checked against the published Random123 known-answer
vectors (and, on the GPU, against curand_Philox4x32_10 in tests/test_gpu_*).
"""
import numpy as np
import pytest
from scipy import stats

import oracle


def gauss(A):
    A = np.asarray(A, np.float64)

    def lg(x):
        return -0.5 * np.sum(A * x * x, axis=1), -A * x
    return lg


def test_leapfrog_gaussian_closed_form():
    A = np.array([0.5, 1.0, 2.0, 3.0])
    x0 = np.array([[1.0, -0.5, 0.3, 2.0]])
    p0 = np.array([[0.2, 0.7, -1.0, 0.1]])
    eps, L = 0.1, 10
    x, p, _, _ = oracle.leapfrog(x0, p0, eps, L, gauss(A))
    for k in range(4):
        a = A[k]
        K = np.array([[1, 0], [-0.5 * eps * a, 1]])   # half kick on (x, p)
        D = np.array([[1, eps], [0, 1]])               # drift
        M = np.linalg.matrix_power(K @ D @ K, L)
        ref = M @ np.array([x0[0, k], p0[0, k]])
        assert x[0, k] == pytest.approx(ref[0], rel=1e-12)
        assert p[0, k] == pytest.approx(ref[1], rel=1e-12)


def test_leapfrog_reversible_and_second_order():
    A = np.array([1.0])
    x0, p0 = np.array([[1.0]]), np.array([[0.0]])
    x, p, _, _ = oracle.leapfrog(x0, p0, 0.2, 25, gauss(A))
    xb, pb, _, _ = oracle.leapfrog(x, -p, 0.2, 25, gauss(A))
    assert xb[0, 0] == pytest.approx(1.0, abs=1e-12) and pb[0, 0] == pytest.approx(0.0, abs=1e-12)
    errs = []
    for eps in (0.1, 0.05):
        x, p, _, _ = oracle.leapfrog(x0, p0, eps, int(round(1.0 / eps)), gauss(A))
        errs.append(abs(0.5 * x[0, 0] ** 2 + 0.5 * p[0, 0] ** 2 - 0.5))
    assert 3.0 < errs[0] / errs[1] < 5.0      # energy error O(ε²)


def test_hmc_moments_standard_normal():
    lg = gauss(np.ones(10))
    C = 64
    x = np.zeros((C, 10))
    draws = []
    acc = []
    for it in range(120):
        x, ap, _, _, _ = oracle.hmc_step(x, 0.3, 8, lg, seed=1234, it=it)
        acc.append(ap.mean())
        if it >= 20:
            draws.append(x.copy())
    d = np.concatenate(draws)
    se = 1.0 / np.sqrt(C * 100 / 3.0)            # generous ESS (autocorrelation)
    assert np.all(np.abs(d.mean(0)) < 3 * se * 3)
    assert np.all(np.abs(d.var(0) - 1.0) < 0.15)
    assert np.mean(acc) > 0.9


def test_hmc_acceptance_to_one_as_eps_to_zero():
    lg = gauss(np.linspace(0.5, 2.0, 6))
    x = np.random.default_rng(0).standard_normal((16, 6))
    _, ap, acc, _, dH = oracle.hmc_step(x, 1e-4, 10, lg, seed=5, it=0)
    assert np.all(ap > 0.9999) and np.all(np.abs(dH) < 1e-6)


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32_10
    assert list(oracle.philox4x32_10([0, 0, 0, 0], [0, 0])) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert list(oracle.philox4x32_10([0xffffffff] * 4, [0xffffffff] * 2)) == \
        [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert list(oracle.philox4x32_10([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                                     [0xa4093822, 0x299f31d0])) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_momenta_are_standard_normal():
    z = np.concatenate([oracle.momenta(2048, 99, 7, c) for c in range(16)])
    assert stats.kstest(z, "norm").pvalue > 1e-3
    assert abs(z.mean()) < 0.03 and abs(z.var() - 1) < 0.04
    u = np.array([oracle.mh_uniform(99, it, 3) for it in range(4000)])
    assert stats.kstest(u, "uniform").pvalue > 1e-3
    # distinct streams per chain / iteration
    assert not np.allclose(oracle.momenta(8, 1, 0, 0), oracle.momenta(8, 1, 0, 1))
    assert not np.allclose(oracle.momenta(8, 1, 0, 0), oracle.momenta(8, 1, 1, 0))


def test_momenta_box_muller_pairs_from_the_raw_philox_words():
    """R22 pairing: parameters 4q, 4q+1 come from Philox words 0, 1 and 4q+2, 4q+3 from
    words 2, 3 of counter (q, chain, iter, 0), key = (seed lo, seed hi), uniforms
    (k + 1/2) 2^-32: each pair's squared radius is -2 ln u(first word) and its angle
    2π u(second word), checked against the raw words of the (known-answer pinned)
    generator; and the four outputs of a counter are uncorrelated (a cos/cos or a
    duplicated pair would give correlation 1)."""
    seed, it, chain, P = 0x0123456789ABCDEF, 5, 3, 4096
    z = oracle.momenta(P, seed, it, chain)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for q in range(0, P // 4, 37):
        w = oracle.philox4x32_10([q, chain, it, 0], key).astype(np.float64)
        u = (w + 0.5) * 2.0 ** -32
        for a in (0, 2):
            z0, z1 = z[4 * q + a], z[4 * q + a + 1]
            assert z0 * z0 + z1 * z1 == pytest.approx(-2.0 * np.log(u[a]), rel=1e-12)
            assert np.mod(np.arctan2(z1, z0), 2 * np.pi) == pytest.approx(2 * np.pi * u[a + 1], abs=1e-9)
    Z = np.concatenate([oracle.momenta(4096, 17, k, 0) for k in range(16)]).reshape(-1, 4)
    cov = np.cov(Z.T)
    se = 1.0 / np.sqrt(len(Z))
    assert np.all(np.abs(cov - np.eye(4)) < 5 * np.sqrt(2) * se), cov


def test_diagonal_mass_is_a_change_of_variables():
    """R19b: HMC / NUTS with diagonal inverse mass m on logp(x) equal the
    identity-mass algorithms (pinned above by closed forms) on y = x / sqrt(m)
    with target logp(sqrt(m) y): momenta q = p sqrt(m), ½ qᵀq = ½ pᵀ M^-1 p,
    velocities M^-1 p in the U-turn criterion."""
    import math
    rng = np.random.default_rng(21)
    P = 6
    A = rng.standard_normal((P, P))
    A = A @ A.T + P * np.eye(P)                       # a correlated Gaussian target
    mu = rng.standard_normal(P)

    def lg(x):
        d = np.atleast_2d(x) - mu
        return -0.5 * np.einsum("ci,ij,cj->c", d, A, d), -(d @ A)
    m = np.array([0.3, 2.0, 1.0, 0.5, 4.0, 0.8])
    sq = np.sqrt(m)

    def lg_y(y):
        lp, g = lg(np.atleast_2d(y) * sq)
        return lp, g * sq
    x0 = rng.standard_normal((3, P))
    p0 = rng.standard_normal((3, P))
    x1, p1, lp1, _ = oracle.leapfrog(x0, p0, 0.05, 7, lg, minv=m)
    y1, q1, lpy, _ = oracle.leapfrog(x0 / sq, p0 * sq, 0.05, 7, lg_y)
    assert np.allclose(x1, y1 * sq, atol=1e-12) and np.allclose(p1 * sq, q1, atol=1e-12)
    seed = 12345
    for it in range(3):
        xa, aa, acca, lpa, dHa = oracle.hmc_step(x0, 0.1, 5, lg, seed, it, minv=m)
        ya, ab, accb, lpb, dHb = oracle.hmc_step(x0 / sq, 0.1, 5, lg_y, seed, it)
        assert np.allclose(xa, ya * sq, atol=1e-12) and np.allclose(dHa, dHb, atol=1e-10)
        assert np.array_equal(acca, accb)
    lg1 = lambda th: (lambda o: (o[0][0], o[1][0]))(lg(th[None]))      # noqa: E731
    lg1y = lambda th: (lambda o: (o[0][0], o[1][0]))(lg_y(th[None]))   # noqa: E731
    for c in range(3):
        lp, g = lg1(x0[c])
        a = oracle.nuts_step(x0[c], lp, g, 0.1, lg1, seed, 5, c, max_depth=5, minv=m)
        lpy0, gy = lg1y(x0[c] / sq)
        b = oracle.nuts_step(x0[c] / sq, lpy0, gy, 0.1, lg1y, seed, 5, c, max_depth=5)
        assert a["depth"] == b["depth"] and a["n_leaves"] == b["n_leaves"]
        assert np.allclose(a["x"], b["x"] * sq, atol=1e-10)
        assert math.isclose(a["accept_stat"], b["accept_stat"], rel_tol=1e-9, abs_tol=1e-12)
