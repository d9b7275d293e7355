"""Exhaustive full-size parity (north_star: "on all five configs"): every ray's
traversal and every distinct chain state of the bench's launches, against the
fp64 oracle, through the C ABI.

  * traversal: the stored (i, j) list of EVERY ray of every geometry (tiny,
    small, medium = configs[2]/[3], ray_sharded = configs[4]) bit-exact, and
    its exit parameters within fp32 rounding (P:234-235 ray, R16 ties);
  * log-posterior / gradient end to end from x (P:225-236, P:403-404 +
    the prior): all 1,024 distinct near-posterior states of configs[2] (the
    1,024-chain launch) and of configs[3] (the 8,192-chain launch, super-chains
    of 8 share a start), the 128 distinct prior-draw states of
    Small and Medium (wide band: worst-case work), and the 16 chains of
    configs[4], each evaluated in the one-chain ray-lanes launch bench.py
    times;
  * determinism (R30): the 8 members of a super-chain get bit-identical logp
    and gradient in the 8,192-chain launch.

Tolerances are north_star's: |Δlogp| <= 1e-4 |logp| and
||Δ∇||_2 <= 1e-3 ||∇||_2 per chain.  Each test records its pass fraction and
worst margin (error / tolerance) in gpurun_out/parity_margins.json.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2603_28907_b200 import Problem, inputs  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEV = "cuda:0"


def record(key, value):
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, "parity_margins.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[key] = value
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def margins(logp_d, grad_d, ref):
    """Per-chain error / tolerance of logp (1e-4 rel) and gradient (1e-3 rel L2)."""
    lp_o, g_o = ref["logp"], ref["grad"]
    e_lp = np.abs(logp_d - lp_o) / np.abs(lp_o) / 1e-4
    e_g = np.linalg.norm(grad_d.astype(np.float64) - g_o, axis=1) / np.linalg.norm(g_o, axis=1) / 1e-3
    return e_lp, e_g


def summarize(key, e_lp, e_g):
    ok = (e_lp <= 1.0) & (e_g <= 1.0)
    s = {"chains": int(ok.size), "pass_fraction": float(ok.mean()),
         "worst_logp_margin": float(e_lp.max()), "worst_grad_margin": float(e_g.max()),
         "median_grad_margin": float(np.median(e_g)), "failing": [int(c) for c in np.nonzero(~ok)[0][:20]]}
    record(key, s)
    return ok, s


@pytest.mark.parametrize("name", ["tiny", "small", "medium", "ray_sharded"])
def test_traversal_every_ray(problems, oracle_problem, name):
    prob = problems(name)
    mp = Problem(prob, device=0, max_chains=1)
    off_d, ij_d, so_d = mp.traversal_all()
    off_o, ij_o, so_o = oracle_problem(name).traversal_all()
    assert np.array_equal(off_d, off_o), "cell counts differ"
    bad = np.nonzero(np.any(ij_d != ij_o, axis=1))[0]
    assert bad.size == 0, f"{bad.size} cells differ, first at ray {np.searchsorted(off_o, bad[0], 'right') - 1}"
    err = np.abs(so_d.astype(np.float64) - so_o)
    assert np.all(err <= 2e-6 * so_o + 1e-5), float((err / (2e-6 * so_o + 1e-5)).max())
    record(f"traversal/{name}", {"rays": int(off_o.size - 1), "cells": int(off_o[-1]), "ij_bit_exact": True,
                                 "worst_s_out_margin": float((err / (2e-6 * so_o + 1e-5)).max())})


def test_all_distinct_near_posterior_states_configs_2_and_3(problems, oracle_problem):
    """configs[2] (1,024 chains) and configs[3] (8,192 chains = 1,024 super-chains of 8,
    the same 1,024 distinct states: chain_states draws one ξ per super-chain) on one
    device, every distinct state against one oracle evaluation of all 1,024."""
    prob, op = problems("medium"), oracle_problem("medium")
    seed = inputs.CONFIGS["medium"].seed
    x1 = inputs.chain_states(prob["x_true"], 1024, seed)
    x8 = inputs.chain_states(prob["x_true"], 8192, seed, super_size=8)
    assert np.array_equal(x8[::8], x1)
    ref = op.logpost_grad(x1.astype(np.float64))
    mp = Problem(prob, device=0, max_chains=8192)
    lp8, g8 = mp.logpost_grad(torch.from_numpy(x8).to(DEV))
    lp8, g8 = lp8.cpu().numpy(), g8.cpu().numpy()
    # R30: identical states in one launch give identical bits
    assert np.array_equal(lp8.reshape(1024, 8), np.repeat(lp8[::8, None], 8, 1))
    assert np.array_equal(g8.reshape(1024, 8, -1), np.repeat(g8[::8, None], 8, 1))
    ok8, s8 = summarize("e2e/configs3_8192", *margins(lp8[::8], g8[::8], ref))
    del mp
    mp = Problem(prob, device=0, max_chains=1024)
    lp1, g1 = mp.logpost_grad(torch.from_numpy(x1).to(DEV))
    ok1, s1 = summarize("e2e/configs2_1024", *margins(lp1.cpu().numpy(), g1.cpu().numpy(), ref))
    assert ok1.all(), s1
    assert ok8.all(), s8


@pytest.mark.parametrize("name,C", [("small", 128), ("medium", 1024)])
def test_all_distinct_prior_draw_states(problems, oracle_problem, name, C):
    """The 128 distinct prior-draw states (data/<config>_prior.npz), in a launch of C
    chains (Medium: the bench's 1,024-chain launch with --states prior, 8 copies each)."""
    prob, op = problems(name), oracle_problem(name)
    x = inputs.prior_states(name, C)
    ref = op.logpost_grad(x[:128].astype(np.float64))
    mp = Problem(prob, device=0, max_chains=C)
    lp, g = mp.logpost_grad(torch.from_numpy(x).to(DEV))
    lp, g = lp.cpu().numpy(), g.cpu().numpy()
    oks = []
    for k in range(C // 128):   # every copy of every distinct state
        ok, s = summarize(f"e2e/prior_{name}_{C}_copy{k}", *margins(lp[128 * k:128 * (k + 1)],
                                                                   g[128 * k:128 * (k + 1)], ref))
        oks.append((ok.all(), s))
    assert all(o for o, _ in oks), [s for o, s in oks if not o]


def test_configs4_all_16_chains(problems, oracle_problem):
    """configs[4]: 16 chains run one after another, each in the one-chain ray-lanes launch
    bench.py times (4,194,304 rays, 8,192 parameters)."""
    prob, op = problems("ray_sharded"), oracle_problem("ray_sharded")
    cfg = inputs.CONFIGS["ray_sharded"]
    x = inputs.chain_states(prob["x_true"], 16, cfg.seed)
    ref = op.logpost_grad(x.astype(np.float64))
    mp = Problem(prob, device=0, max_chains=1)
    lp, g = [], []
    for c in range(16):
        a, b = mp.logpost_grad(torch.from_numpy(x[c:c + 1]).to(DEV))
        lp.append(a.cpu().numpy()[0])
        g.append(b.cpu().numpy()[0])
    ok, s = summarize("e2e/configs4_16_chains", *margins(np.array(lp), np.array(g), ref))
    assert ok.all(), s
