"""Posterior summaries (reading R27): oracle pins
(definitions, the [0, 0.5] bound of the indicator std, telescoping of
the indicators, MAP = argmax) and GPU accumulators against the oracle."""
import numpy as np
import pytest

import oracle
from paper_2603_28907_b200 import inputs


def test_indicators_sum_and_bounds():
    rng = np.random.default_rng(0)
    H0 = rng.uniform(50, 150, (4, 5))
    H1 = H0 + rng.uniform(1, 80, (4, 5))
    D = oracle.layer_indicators(H0, H1, 300.0, 30)
    z = np.arange(30) * 10.0
    assert np.allclose(D.sum(0), oracle.sigmoid(300.0 - z) - oracle.sigmoid(-z))   # telescoping
    assert D.min() >= 0 and D.max() <= 1       # D in [0, 1), 1 by fp64 saturation
    # far from the interfaces the indicators are the Heaviside layer map
    k = 0
    assert np.allclose(D[0, ..., 20], 0, atol=1e-6) and np.all(D[2, ..., 29] > 0.99)


def test_summaries_definitions(problems):
    op = oracle.Problem(problems("tiny"))
    x = inputs.chain_states(op.prob["x_true"], 3, 1, scale=0.3).astype(np.float64)
    one = oracle.posterior_summaries(op, [x[:1]], [np.array([-5.0])], 12, 10.0)
    assert np.allclose(one["mean_heights"], op.heights(x[0])[0])
    assert np.all(one["indicator_std"] == 0)
    s = oracle.posterior_summaries(op, [x], [np.array([-5.0, -3.0, -3.0])], 12, 10.0)
    assert s["map_logp"] == -3.0 and np.array_equal(s["map_x"], x[1])      # argmax, first of ties
    assert s["indicator_std"].max() <= 0.5 + 1e-12
    # two draws whose muck top differs by far more than γ: the indicator of a voxel
    # between them is ~0 in one draw and ~1 in the other -> std ~ 0.5
    H = op.heights(x[0])[0]
    lo = op.latent_from_heights(np.stack([H[0] * 0 + 60.0, H[1]]))
    hi = op.latent_from_heights(np.stack([H[0] * 0 + 140.0, H[1]]))
    s2 = oracle.posterior_summaries(op, [np.stack([lo, hi])], [np.zeros(2)], 30, 10.0)
    assert s2["indicator_std"][0, :, :, 10].min() > 0.49        # z = 100 m


@pytest.mark.gpu
def test_summary_accumulators_match_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_28907_b200 import Problem
    prob = inputs.make_problem("small")
    op = oracle.Problem(prob)
    mp = Problem(prob, device=0, max_chains=16)
    nz, gap = 24, 12.0
    acc, map_x, map_lp = mp.summary_buffers(nz)
    draws, lps = [], []
    for it in range(3):
        x = inputs.chain_states(prob["x_true"], 16, 7 + it, scale=0.2)
        xt = torch.from_numpy(x).cuda()
        lp, _ = mp.logpost_grad(xt)
        mp.summary_update(xt, lp, acc, nz, gap, map_x, map_lp)
        draws.append(x)
        lps.append(lp.cpu().numpy())
    s = mp.summaries(acc, nz)
    ref = oracle.posterior_summaries(op, draws, lps, nz, gap)
    assert s["draws"] == ref["draws"] == 48
    assert np.allclose(s["mean_heights"], ref["mean_heights"], rtol=1e-6)
    assert np.array_equal(s["gap_probability"], ref["gap_probability"])
    assert np.allclose(s["indicator_std"], ref["indicator_std"], atol=2e-5)
    assert float(map_lp.cpu()[0]) == pytest.approx(ref["map_logp"], rel=1e-12)
    assert np.allclose(map_x.cpu().numpy(), ref["map_x"], atol=1e-6)
