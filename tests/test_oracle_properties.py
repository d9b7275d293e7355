"""Property tests (hypothesis) of the oracle on random geometries, SURVEY §4:
partition of every ray's in-box length into muck / air / rock, non-negative
lengths, opacity monotone in each surface's heights, the copula marginal
ǔ = Φ(x/σ) uniform under the CAR prior (a KS test), and the voxel
lengths partition (f3)."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st
from scipy import stats

import oracle

SETTINGS = dict(max_examples=12, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.function_scoped_fixture])


def random_heights(rng, n, z_top=300.0, rough=1.0):
    """Ordered bilinear surfaces 0 < H0 < H1 < z_top, smooth (rough=0) to rough (1)."""
    base0 = rng.uniform(60, 160)
    H0 = base0 + rough * rng.normal(0, 25, (n, n))
    H1 = H0 + rng.uniform(1, 60) + rough * np.abs(rng.normal(0, 20, (n, n)))
    return np.clip(np.stack([H0, H1]), 0.5, z_top - 0.5)


@settings(**SETTINGS)
@given(seed=st.integers(0, 2 ** 31 - 1), rough=st.floats(0.0, 1.0))
def test_lengths_partition_and_are_nonnegative(oracle_problem, seed, rough):
    op = oracle_problem("tiny")
    H = random_heights(np.random.default_rng(seed), op.nx, rough=rough)
    L, O = op.path_lengths(H[None])
    s_exit = np.array([op.ray_extent(q)[0] for q in range(op.R)])
    assert np.all(L >= -1e-9)
    assert np.allclose(L[0].sum(1), s_exit, rtol=1e-12, atol=1e-9)


@settings(**SETTINGS)
@given(seed=st.integers(0, 2 ** 31 - 1), node=st.integers(0, 63), surf=st.integers(0, 1),
       dh=st.floats(0.01, 5.0))
def test_opacity_monotone_in_heights(oracle_problem, seed, node, surf, dh):
    """ρ_m > ρ_a < ρ_r: raising a muck-top node never lowers the opacity, raising a
    cave-back node never raises it (∂B/∂h >= 0)."""
    op = oracle_problem("tiny")
    H = random_heights(np.random.default_rng(seed), op.nx)
    Hp = H.copy()
    i, j = divmod(node, op.ny)
    Hp[surf, i, j] += dh
    if surf == 0:
        Hp[1, i, j] = max(Hp[1, i, j], Hp[0, i, j] + 0.1)
        if Hp[1, i, j] != H[1, i, j]:
            return                                     # both surfaces moved: no sign claim
    _, O0 = op.path_lengths(H[None])
    _, O1 = op.path_lengths(Hp[None])
    d = O1[0] - O0[0]
    if surf == 0:
        assert np.all(d >= -1e-9)
    else:
        assert np.all(d <= 1e-9)


@settings(**SETTINGS)
@given(q=st.integers(0, 16383), nz=st.integers(1, 80))
def test_voxel_lengths_partition(oracle_problem, q, nz):
    op = oracle_problem("small")
    vox, ln = op.voxel_path(nz, q)
    assert np.all(ln > 0) and np.all((vox >= 0) & (vox < op.N * nz))
    assert ln.sum() == pytest.approx(op.ray_extent(q)[0], rel=1e-12)
    assert len(set(vox.tolist())) == len(vox)              # every piece in a different voxel


def test_copula_marginal_is_uniform_under_the_prior(oracle_problem):
    """x ~ N(0, Q^-1) on the torus and ǔ = Φ(x/σ) with σ² = Σ_ii: every
    ǔ_i is Unif(0,1) (KS test on one node over many prior draws)."""
    op = oracle_problem("small")
    rng = np.random.default_rng(8)
    sig = op.sigma()
    x0 = oracle.prior_draws(op.nx, op.ny, op.car_r[0], 4000, rng)[:, 37]
    u = stats.norm.cdf(x0 / sig[0])
    assert stats.kstest(u, "uniform").pvalue > 1e-3
    # and through the oracle's own heights map: H0 / z_top = ǔ0
    x = np.zeros(op.P)
    x[:op.N] = oracle.prior_draws(op.nx, op.ny, op.car_r[0], 1, rng)[0]
    H, _ = op.heights(x)
    assert np.allclose(H[0].reshape(-1) / op.z_top, stats.norm.cdf(x[:op.N] / sig[0]), rtol=1e-12)
