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
