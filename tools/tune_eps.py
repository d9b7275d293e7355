"""Tune the HMC step size by the warm-up protocol (reading R20) and store it.

Runs dual averaging (target acceptance 0.8) for the config's warm-up length
(BASELINE configs[3]: 100 of 200 iterations) on the GPU path from the
near-posterior start, then a few sampling iterations at the final ε, and
writes data/tuned_eps.json {config: {eps, warmup_iters, mean_accept_sampling}}.
bench.py times sampling-phase iterations at this ε (a stationary workload),
instead of the first iterations of dual averaging, whose early steps inflate ε
by orders of magnitude by design.

  python tools/tune_eps.py [config] [--chains C] [--warmup 100] [--sample 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2603_28907_b200 import Problem, inputs  # noqa: E402
from paper_2603_28907_b200.hmc import ChainShard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="medium")
    ap.add_argument("--chains", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--sample", type=int, default=10)
    a = ap.parse_args()
    cfg = inputs.CONFIGS[a.config]
    C = a.chains or min(cfg.chains, 1024)
    prob = inputs.make_problem(a.config)
    pb = Problem(prob, device=0, max_chains=C)
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed, super_size=8)
    sh = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=cfg.leapfrog_steps, eps0=cfg.eps)
    acc = [sh.step(adapt=True) for _ in range(a.warmup)]
    sh.end_warmup()
    eps = float(sh.eps[0])
    acc_s = []
    for _ in range(a.sample):
        sh.step(adapt=False, sample=True)
        acc_s.append(float(sh.acc_prob.mean()))
    path = os.path.join(inputs.DATA_DIR, "tuned_eps.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[a.config] = {"eps": eps, "warmup_iters": a.warmup, "chains": C,
                      "mean_accept_last_warmup": float(np.mean(acc[-10:])),
                      "mean_accept_sampling": float(np.mean(acc_s))}
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(a.config, json.dumps(data[a.config]))


if __name__ == "__main__":
    main()
