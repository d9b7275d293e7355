"""Pins for the oracle NUTS (reading R26): the iterative U-turn
checkpoints against the recursive definition (every aligned power-of-two
sub-trajectory is checked exactly once, when its last leaf is built),
sampling a 10-D standard normal (moments within Monte Carlo error), and the
small-step limits (acceptance -> 1; the trajectory grows until it turns back
after about half a period, π/ε steps, of the harmonic oscillator)."""
import math

import numpy as np
import pytest

import oracle


def test_iterative_checkpoints_check_every_aligned_subtree_once():
    for j in range(1, 9):
        owner = {}
        checked = set()
        for n in range(2 ** j):
            lo, hi = oracle.leaf_ckpt_idxs(n)
            if n % 2 == 0:
                owner[hi] = n
            else:
                for i in range(hi, lo - 1, -1):
                    checked.add((owner[i], n))
        want = {(s, s + 2 ** k - 1) for k in range(1, j + 1) for s in range(0, 2 ** j, 2 ** k)}
        assert checked == want, j


def test_is_turning_matches_definition():
    rng = np.random.default_rng(0)
    for _ in range(200):
        a, b, r = rng.standard_normal((3, 5))
        rs = r - 0.5 * (a + b)
        assert oracle.is_turning(a, b, r) == (a @ rs <= 0 or b @ rs <= 0)


def std_normal(x):
    return -0.5 * float(x @ x), -x


def test_nuts_moments_standard_normal():
    D, n = 10, 1500
    x = np.zeros(D)
    lp, g = std_normal(x)
    xs, depths = [], []
    for it in range(n):
        out = oracle.nuts_step(x, lp, g, 0.35, std_normal, 0x1234, it, 0, max_depth=6)
        x, lp, g = out["x"], out["logp"], out["grad"]
        xs.append(x)
        depths.append(out["depth"])
    xs = np.array(xs[100:])
    se = 1.0 / math.sqrt(len(xs))      # NUTS draws of a Gaussian are nearly independent
    assert np.all(np.abs(xs.mean(0)) < 5 * se)
    assert np.all(np.abs(xs.var(0) - 1.0) < 8 * se * math.sqrt(2))
    assert 2 <= np.mean(depths) <= 5


def test_nuts_small_step_limits():
    D = 4
    x = np.full(D, 0.5)
    lp, g = std_normal(x)
    eps = 0.01
    out = oracle.nuts_step(x, lp, g, eps, std_normal, 99, 0, 0, max_depth=12)
    assert out["accept_stat"] > 0.999 and not out["diverging"]
    # a harmonic trajectory turns back after ~π/ε steps: the doubling stops at the
    # first depth whose tree spans more than that
    assert 2 ** (out["depth"] - 1) <= 2 * math.pi / eps and 2 ** out["depth"] >= math.pi / (2 * eps)
