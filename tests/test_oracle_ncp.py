"""Oracle pins for the non-centred CAR parameterisation x = U z (
SURVEY §8(f) f2; reading R13d in DESIGN.md).

Pinned against: U² = Q(r)^{-1} and dU/dr from dense numpy matrices built from
the definition (Q = diag(A1) - rA; U by numpy's symmetric eigendecomposition);
the already-pinned centred oracle at x = U z (same likelihood, same σ); the
standard-normal log density of z (scipy); central finite differences in z and ρ.
"""
import numpy as np
import pytest
from scipy.stats import logistic, norm

import oracle
from paper_2603_28907_b200 import inputs
from test_oracle_prior import dense_Q


def circulant(k):
    nx, ny = k.shape
    N = nx * ny
    M = np.zeros((N, N))
    for i in range(nx):
        for j in range(ny):
            for i2 in range(nx):
                for j2 in range(ny):
                    M[i * ny + j, i2 * ny + j2] = k[(i - i2) % nx, (j - j2) % ny]
    return M


def sym_sqrt_inv(Q):
    w, V = np.linalg.eigh(Q)
    return (V / np.sqrt(w)) @ V.T


@pytest.mark.parametrize("nx,ny,r", [(4, 4, 0.8), (3, 5, 0.95), (6, 4, 0.3)])
def test_U_is_the_symmetric_root_of_the_covariance(nx, ny, r):
    k, dk = oracle.ncp_kernel(nx, ny, r)
    U = circulant(k)
    Q = dense_Q(nx, ny, r)
    assert np.allclose(U @ U, np.linalg.inv(Q), atol=1e-12)        # Σ = U Uᵀ
    assert np.allclose(U, sym_sqrt_inv(Q), atol=1e-12)
    h = 1e-6
    dU = (sym_sqrt_inv(dense_Q(nx, ny, r + h)) - sym_sqrt_inv(dense_Q(nx, ny, r - h))) / (2 * h)
    assert np.allclose(circulant(dk), dU, atol=1e-8)


def _ncp_state(prob, op, C, seed, rho):
    """Non-centred states whose x = U z are the near-posterior centred states."""
    x = inputs.chain_states(prob["x_true"], C, seed, scale=0.05).astype(np.float64)
    v = np.zeros((C, op.P + 2))
    for l in range(2):
        r = 1.0 / (1.0 + np.exp(-rho[l]))
        U = circulant(oracle.ncp_kernel(op.nx, op.ny, r)[0])
        v[:, l * op.N:(l + 1) * op.N] = np.linalg.solve(U, x[:, l * op.N:(l + 1) * op.N].T).T
        v[:, 2 * op.N + l] = rho[l]
    return v, x


def test_ncp_matches_the_centred_model_at_x_equal_Uz(problems, oracle_problem):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    rho = (2.5, 2.0)
    v, x = _ncp_state(prob, op, 3, 1, rho)
    out = op.logpost_grad_ncp(v)
    cen = op.logpost_grad_r(np.concatenate([x, np.broadcast_to(rho, (3, 2))], axis=1))
    assert np.allclose(out["ll_dev"], cen["ll_dev"], rtol=1e-12)      # same heights, same σ(r)
    z = v[:, :op.P]
    ref = out["ll_dev"] + norm.logpdf(z).sum(1) + logistic.logpdf(np.asarray(rho)).sum()
    assert np.allclose(out["logp"], ref, rtol=1e-12)


def test_ncp_gradient_vs_fd(problems, oracle_problem):
    prob = problems("tiny")
    op = oracle_problem("tiny")
    v, _ = _ncp_state(prob, op, 2, 1, (2.5, 1.5))
    out = op.logpost_grad_ncp(v)
    rng = np.random.default_rng(4)
    ks = list(rng.choice(op.P, 16, replace=False)) + [op.P, op.P + 1]
    for c in range(2):
        for k in ks:
            h = 1e-6 if k < op.P else 1e-5
            vp, vm = v.copy(), v.copy()
            vp[c, k] += h
            vm[c, k] -= h
            fd = (op.logpost_grad_ncp(vp[c:c + 1])["logp"][0] - op.logpost_grad_ncp(vm[c:c + 1])["logp"][0]) / (2 * h)
            assert out["grad"][c, k] == pytest.approx(fd, rel=2e-5, abs=1e-3)


def test_noncentred_state_helper_inverts_U():
    """hmc.noncentred_state (host helper for starting non-centred chains) gives
    U(r) z = x with the oracle's U (dense circulant)."""
    from paper_2603_28907_b200.hmc import noncentred_state
    nx, ny, rho = 3, 4, (1.0, 2.0)
    x = np.random.default_rng(0).standard_normal((2, 2 * nx * ny))
    v = noncentred_state(x, rho, nx, ny).astype(np.float64)
    N = nx * ny
    for l in range(2):
        U = circulant(oracle.ncp_kernel(nx, ny, 1 / (1 + np.exp(-rho[l])))[0])
        assert np.allclose(v[:, l * N:(l + 1) * N] @ U.T, x[:, l * N:(l + 1) * N], atol=1e-6)
        assert np.all(v[:, 2 * N + l] == np.float32(rho[l]))
