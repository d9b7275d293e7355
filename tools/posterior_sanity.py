"""Posterior sanity on Small (SURVEY §8(c.3) "internal sanity only"): the mean
heights after warm-up vs the synthetic truth over the central (ray-covered)
nodes, from prior draws or from near-truth starts (x_true + 0.05 ξ).

  python tools/posterior_sanity.py [n_warmup] [n_sample] [prior|near]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2603_28907_b200 import Problem, inputs  # noqa: E402
from paper_2603_28907_b200.hmc import ChainShard  # noqa: E402


def main():
    nw = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    start = sys.argv[3] if len(sys.argv) > 3 else "prior"   # prior | near
    prob = inputs.make_problem("small")
    cfg = inputs.CONFIGS["small"]
    C = 64
    mp = Problem(prob, device=0, max_chains=C)
    x0 = (inputs.prior_states("small", C) if start == "prior"
          else inputs.chain_states(prob["x_true"], C, cfg.seed, scale=0.05))
    H0 = mp.heights(torch.from_numpy(x0).cuda()).cpu().numpy()
    sh = ChainShard(mp, x0, seed=inputs.philox_key(cfg), L=10, eps0=1e-3)
    out = sh.run(nw, ns)
    H = mp.heights(sh.x).cpu().numpy()
    Ht = prob["H_true"]
    mask = np.zeros(Ht.shape[1:], bool)          # central nodes (inside the detectors' cones)
    n = Ht.shape[1]
    mask[n // 4:3 * n // 4, n // 4:3 * n // 4] = True
    e0 = np.abs(H0.mean(0) - Ht)[:, mask].mean(1)
    e1 = np.abs(H.mean(0) - Ht)[:, mask].mean(1)
    sd = H.std(0)[:, mask].mean(1)
    print(json.dumps({"start": start, "warmup": nw, "sample": ns, "across_chain_sd_m": sd.tolist(), "final_eps": float(sh.eps[0]),
                      "accept_last": float(np.mean(out["warmup_accept"][-10:])),
                      "mean_abs_err_start_m": e0.tolist(), "mean_abs_err_end_m": e1.tolist(),
                      "rhat_max": float(np.max(out["rhat"]))}))


if __name__ == "__main__":
    main()
