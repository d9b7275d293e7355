"""Nested R̂ (reading R21b; SPEC's decomposition used for test ideas
only): host assembly from partial sums against a direct numpy computation from
the draws, the calibration / separated-mode behaviour, and (GPU) the partial-sum
kernel against numpy."""
import numpy as np
import pytest

from paper_2603_28907_b200.hmc import nested_rhat_from_partials


def nested_rhat_direct(draws, M):
    """draws [n_draw][C][P] -> nested R̂ [P], chains [kM, (k+1)M) = super-chain k:
    B = unbiased variance of super-chain means, W = mean over super-chains of
    (mean within-chain variance + variance of the chain means within it)."""
    n, C, P = draws.shape
    K = C // M
    d = draws.reshape(n, K, M, P)
    chain_mean = d.mean(0)                                   # [K][M][P]
    wt = d.var(0, ddof=1).mean(1) if n > 1 else np.zeros((K, P))
    bt = chain_mean.var(1, ddof=1) if M > 1 else np.zeros((K, P))
    m_k = chain_mean.mean(1)
    B = m_k.var(0, ddof=1)
    W = (wt + bt).mean(0)
    return np.sqrt(1 + B / W)


def partials_numpy(draws, M):
    n, C, P = draws.shape
    K = C // M
    d = draws.reshape(n, K, M, P)
    chain_mean = d.mean(0)
    wt = d.var(0, ddof=1).mean(1) if n > 1 else np.zeros((K, P))
    bt = chain_mean.var(1, ddof=1) if M > 1 else np.zeros((K, P))
    m_k = chain_mean.mean(1)
    return np.stack([m_k.sum(0), (m_k ** 2).sum(0), (wt + bt).sum(0)]), K


@pytest.mark.parametrize("n,M", [(1, 8), (20, 4), (5, 1)])
def test_assembly_matches_direct(n, M):
    rng = np.random.default_rng(n * 10 + M)
    draws = rng.standard_normal((n, 64, 7)) + rng.standard_normal((1, 64, 7)) * 0.3
    part, K = partials_numpy(draws, M)
    assert np.allclose(nested_rhat_from_partials(part, K), nested_rhat_direct(draws, M), rtol=1e-12)


@pytest.mark.parametrize("M", [4, 8])
def test_calibration_and_separated_modes(M):
    # iid N(0,1) keep-last draws, K = 8 super-chains: B estimates σ²/M and W
    # estimates σ², so R̂² - 1 centres on 1/M (with M = 8 as in the paper, P:689-691,
    # R̂ ≈ 1.06; its worst reported value is 1.12)
    rng = np.random.default_rng(5)
    vals = [nested_rhat_direct(rng.standard_normal((1, 8 * M, 1)), M)[0] ** 2 - 1 for _ in range(400)]
    assert 0.6 / M < np.median(vals) < 1.4 / M
    d = rng.standard_normal((1, 8 * M, 1)) + np.repeat(10.0 * np.arange(8), M)[None, :, None]
    assert nested_rhat_direct(d, M)[0] > 2


@pytest.mark.gpu
def test_nested_partials_kernel_matches_numpy():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_28907_b200 import Problem, inputs
    mp = Problem(inputs.make_problem("small"), device=0, max_chains=64)
    rng = np.random.default_rng(2)
    for n, M in ((1, 8), (12, 8), (12, 4)):
        draws = (rng.standard_normal((n, 64, mp.P)) + rng.standard_normal((1, 64, mp.P))).astype(np.float32)
        mean = torch.zeros((64, mp.P), device="cuda")
        m2 = torch.zeros((64, mp.P), device="cuda")
        for it in range(n):
            mp.stats_update(64, x=torch.from_numpy(draws[it]).cuda(), n_prev=it, mean=mean, m2=m2)
        part = mp.nested_rhat_partials(64, M, mean, m2, n).cpu().numpy()
        ref, K = partials_numpy(draws.astype(np.float64), M)
        assert np.allclose(part, ref, rtol=2e-4, atol=1e-3)
        assert np.allclose(nested_rhat_from_partials(part, K), nested_rhat_direct(draws.astype(np.float64), M),
                           rtol=1e-3)
