"""Oracle pins: CAR prior on the torus and the latent -> heights map.

Each pin checks the oracle against something other than itself: a dense
precision matrix built here from the paper's definition (P:513-535,
P:551-557) and a library routine (numpy inv/slogdet, scipy mvn logpdf, ndtr),
closed forms the paper fixes, or central finite differences.
"""
import math

import numpy as np
import pytest
from scipy.special import ndtr
from scipy.stats import multivariate_normal

import oracle


def torus_adjacency(nr, nc):
    """A_ij = 1 iff i ~ j on the periodic nearest-neighbour grid (Fig. 7)."""
    N = nr * nc
    A = np.zeros((N, N))
    for i in range(nr):
        for j in range(nc):
            a = i * nc + j
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                b = ((i + di) % nr) * nc + (j + dj) % nc
                A[a, b] = 1.0
    return A


def dense_Q(nr, nc, r):
    A = torus_adjacency(nr, nc)
    return np.diag(A @ np.ones(len(A))) - r * A


def test_adjacency_matches_paper_figure():
    # P:540-549 (Fig. 7): neighbourhoods wrap around the edges of a 12x15 grid
    A = torus_adjacency(12, 15)
    nb = {divmod(int(k), 15) for k in np.nonzero(A[0])[0]}
    assert nb == {(11, 0), (1, 0), (0, 14), (0, 1)}
    # 3x3 torus: 9 nodes, 18 edges, every degree 4
    A3 = torus_adjacency(3, 3)
    assert A3.sum() / 2 == 18 and np.all(A3.sum(1) == 4) and np.all(np.diag(A3) == 0)


def test_Q_textbook_facts():
    for r in (0.0, 0.5, 0.95):
        Q = dense_Q(4, 5, r)
        assert np.allclose(Q @ np.ones(20), (4 - 4 * r) * np.ones(20))   # row sums
        assert np.linalg.eigvalsh(Q).min() > 0                            # PD
    assert np.array_equal(dense_Q(3, 3, 0.0), 4 * np.eye(9))
    # full conditionals: E[x_i|x_-i] = (r/4) Σ_j x_j, Var = 1/4
    r = 0.8
    Q = dense_Q(4, 4, r)
    x = np.random.default_rng(0).standard_normal(16)
    i = 5
    cond_mean = -(Q[i] @ x - Q[i, i] * x[i]) / Q[i, i]
    assert cond_mean == pytest.approx(r / 4 * (torus_adjacency(4, 4)[i] @ x), rel=1e-14)
    assert 1.0 / Q[i, i] == 0.25


@pytest.mark.parametrize("nr,nc,r", [(3, 3, 0.5), (4, 4, 0.8), (4, 6, 0.95), (8, 8, 0.95), (5, 7, 0.0)])
def test_torus_spectrum_vs_dense(nr, nc, r):
    Q = dense_Q(nr, nc, r)
    S = np.linalg.inv(Q)
    sigma, logdet = oracle.torus_spectrum(nr, nc, r)
    assert np.allclose(np.diag(S), sigma ** 2, rtol=1e-12)   # equal marginals
    assert logdet == pytest.approx(np.linalg.slogdet(Q)[1], rel=1e-12)


def test_torus_spectrum_survey_values():
    # SURVEY.md Appendix A (closed form checked against a dense inverse)
    s, ld = oracle.torus_spectrum(4, 4, 0.8)
    assert s ** 2 == pytest.approx(0.3293650794, rel=1e-9)
    assert ld == pytest.approx(20.461645, rel=1e-7)
    assert oracle.torus_spectrum(8, 8, 0.95)[0] == pytest.approx(0.6524405203, rel=1e-9)
    assert oracle.torus_spectrum(32, 32, 0.95)[0] == pytest.approx(0.6420383109, rel=1e-9)
    assert oracle.torus_spectrum(3, 3, 0.0)[0] == 0.5


@pytest.mark.parametrize("nr,nc,r", [(3, 3, 0.3), (4, 5, 0.8), (6, 6, 0.95)])
def test_prior_value_and_gradient(nr, nc, r):
    Q = dense_Q(nr, nc, r)
    rng = np.random.default_rng(nr * nc)
    x = rng.standard_normal((nr, nc))
    v, g = oracle.prior_surface(x, r)
    ref = multivariate_normal(mean=np.zeros(nr * nc), cov=np.linalg.inv(Q)).logpdf(x.ravel())
    assert v == pytest.approx(ref, rel=1e-11)
    assert np.allclose(g.ravel(), -Q @ x.ravel(), rtol=1e-13, atol=1e-13)
    # central FD on the value
    h = 1e-5
    for k in range(0, nr * nc, 3):
        e = np.zeros(nr * nc)
        e[k] = h
        fd = (oracle.prior_surface((x.ravel() + e).reshape(nr, nc), r)[0]
              - oracle.prior_surface((x.ravel() - e).reshape(nr, nc), r)[0]) / (2 * h)
        assert fd == pytest.approx(g.ravel()[k], rel=1e-7, abs=1e-8)


# --------------------------------------------------------------------------
# heights map
# --------------------------------------------------------------------------

def test_heights_closed_forms(oracle_problem):
    op = oracle_problem("tiny")
    zt = op.z_top
    H, _ = op.heights(np.zeros(op.P))
    # ǔ = Φ(0) = 1/2 -> H_1 = z_top/2, H_2 = (1/2)(z_top/2) + (1/2) z_top = 3/4 z_top (S:333-334 scaled)
    assert np.all(H[0] == 0.5 * zt) and np.allclose(H[1], 0.75 * zt, rtol=1e-15)
    s = op.sigma()
    x = np.concatenate([np.full(op.N, s[0]), np.zeros(op.N)])
    H, _ = op.heights(x)
    assert np.allclose(H[0], ndtr(1.0) * zt, rtol=1e-15)
    assert ndtr(1.0) == pytest.approx(0.8413447, abs=1e-7)
    assert np.allclose(H[1], H[0] + 0.5 * (zt - H[0]), rtol=1e-15)


def test_heights_ordered_and_fd(oracle_problem):
    op = oracle_problem("tiny")
    rng = np.random.default_rng(3)
    sg = np.repeat(op.sigma(), op.N)
    for _ in range(20):
        # strict ordering holds while Φ(t) < 1 in fp64; |t| <= 5 covers the prior mass
        x = sg * np.clip(1.5 * rng.standard_normal(op.P), -5, 5)
        H, dH = op.heights(x)
        assert np.all(H[0] > 0) and np.all(H[1] > H[0]) and np.all(H[1] < op.z_top)
    H, _ = op.heights(sg * 10.5 * rng.choice([-1.0, 1.0], op.P))
    assert np.all(H[0] >= 0) and np.all(H[1] >= H[0]) and np.all(H[1] <= op.z_top)
    x = rng.standard_normal(op.P) * 0.5
    H, dH = op.heights(x)
    h = 1e-6
    N = op.N
    for k in (0, 7, 33):
        for l in (0, 1):
            e = np.zeros(op.P)
            e[l * N + k] = h
            Hp, _ = op.heights(x + e)
            Hm, _ = op.heights(x - e)
            d = (Hp - Hm).reshape(2, N)[:, k] / (2 * h)
            if l == 0:
                assert d[0] == pytest.approx(dH[0].ravel()[k], rel=1e-7)
                assert d[1] == pytest.approx(dH[1].ravel()[k], rel=1e-7)
            else:
                assert d[0] == 0.0
                assert d[1] == pytest.approx(dH[2].ravel()[k], rel=1e-7)


def test_heights_clamp_and_inverse(oracle_problem):
    op = oracle_problem("small")
    s = op.sigma()
    x = np.zeros(op.P)
    x[0] = 11 * s[0]
    x[op.N] = -11 * s[1]
    _, dH = op.heights(x)
    assert dH[0].ravel()[0] == 0.0 and dH[2].ravel()[0] == 0.0      # R18
    xt = op.prob["x_true"]
    H, _ = op.heights(xt)
    assert np.allclose(H, op.prob["H_true"], rtol=1e-12, atol=1e-9)
    assert np.allclose(op.latent_from_heights(H), xt, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("nr,nc,r", [(4, 4, 0.8), (3, 5, 0.95)])
def test_prior_draws_covariance(nr, nc, r):
    """oracle.prior_draws (the prior-draw chain states of SURVEY §8(d.1)) has
    covariance Q^-1 (dense numpy inverse of the definition) and E[xᵀQx] = N."""
    rng = np.random.default_rng(17)
    n = 200000
    x = oracle.prior_draws(nr, nc, r, n, rng)
    Qi = np.linalg.inv(dense_Q(nr, nc, r))
    emp = x.T @ x / n
    se = np.sqrt((Qi ** 2 + np.outer(np.diag(Qi), np.diag(Qi))) / n)   # MC s.e. of a Gaussian covariance
    assert np.all(np.abs(emp - Qi) < 5 * se)
    quad = np.einsum("ni,ij,nj->n", x, dense_Q(nr, nc, r), x)
    assert abs(quad.mean() - nr * nc) < 5 * np.sqrt(2 * nr * nc / n)
