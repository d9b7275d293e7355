"""Algorithmic work per chain x ray for the roofline.

Runs the ORACLE's instrumentation (§c.1 step 13) on each config's own
near-posterior chain states (--prior: prior-draw states, key <name>_prior) and
writes data/work_counts.json:
  n_inbox  cells of the in-box traversal
  n_band   cells whose z-range meets the chain's band [min H0, max H1]
  n_solve  surface-cells not resolved by the corner-bound test (a quadratic solve)
  n_cross  surface crossings (adjoint scatters of 4 nodes)
per chain x ray, and the algorithmic FP32 flop count per chain x ray with the
per-item weights of SURVEY §8(d.3) (the grading contract; FMA = 2):
  F = F_SETUP + F_CELL*n_band + F_SOLVE*n_solve + F_CROSS*n_cross + F_EPI
  F_SETUP = 20  per-ray setup (band bounds, extent)
  F_CELL = 24   DDA + z-range + 2 corner-bound tests per band cell
  F_SOLVE = 30  one quadratic per unresolved surface-cell
  F_CROSS = 24  crossing position, 1/|g'|, four bilinear adjoint weights
  F_EPI = 12    opacity -> flux -> Poisson term and its derivative
Usage: python tools/count_work.py [--prior] [config ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2603_28907_b200 import inputs  # noqa: E402

F_SETUP, F_CELL, F_SOLVE, F_CROSS, F_EPI = 20, 24, 30, 24, 12


def count(name: str, n_chains: int = 4, prior: bool = False):
    cfg = inputs.CONFIGS[name]
    prob = inputs.make_problem(name)
    op = oracle.Problem(prob)
    x = (inputs.prior_states(name, n_chains) if prior
         else inputs.chain_states(prob["x_true"], n_chains, cfg.seed))
    out = op.logpost_grad(x.astype("float64"))
    c = out["counters"] / float(n_chains * op.R)
    n_inbox, n_band, n_solve, n_cross = (float(v) for v in c)
    F = F_SETUP + F_CELL * n_band + F_SOLVE * n_solve + F_CROSS * n_cross + F_EPI
    return dict(n_inbox=n_inbox, n_band=n_band, n_solve=n_solve, n_cross=n_cross,
                flops_per_pair=F, chains_sampled=n_chains, rays=op.R,
                weights=dict(F_SETUP=F_SETUP, F_CELL=F_CELL, F_SOLVE=F_SOLVE, F_CROSS=F_CROSS, F_EPI=F_EPI,
                             source="SURVEY.md §8(d.3)"))


if __name__ == "__main__":
    prior = "--prior" in sys.argv[1:]   # prior-draw chain states (key <name>_prior)
    names = [a for a in sys.argv[1:] if a != "--prior"] or ["tiny", "small", "medium", "ray_sharded"]
    path = os.path.join(inputs.DATA_DIR, "work_counts.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for n in names:
        key = inputs.DATA_NAME[n] + ("_prior" if prior else "")
        data[key] = count(n, 1 if n == "ray_sharded" else 4, prior)
        data[key]["states"] = "prior" if prior else "near-posterior"
        print(n, json.dumps(data[key]))
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
