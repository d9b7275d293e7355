"""Locate the rays behind a trace/adjoint discrepancy (test infrastructure).

For one chain's fp32 heights (the device's), evaluate ∂ℓ/∂H on ray subsets with
both the device (mt_loglik_heights) and the fp64 oracle fed the same fp32
heights, and recursively split the subsets whose error is large, down to single
rays; print those rays with their per-ray discrepancy and geometry.

  python tools/ray_bisect.py <config> <chain> [--prior] [--min 1e-3]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs  # noqa: E402


def sub(prob, idx):
    p = dict(prob)
    for k in ("ray_det", "ray_dir", "ray_w", "counts"):
        p[k] = np.ascontiguousarray(np.asarray(prob[k])[idx])
    return p


def main():
    name, chain = sys.argv[1], int(sys.argv[2])
    prior = "--prior" in sys.argv
    cfg = inputs.CONFIGS[name]
    prob = inputs.make_problem(name)
    x = (inputs.prior_states(name, chain + 1) if prior else inputs.chain_states(prob["x_true"], chain + 1, cfg.seed))[chain:chain + 1]
    mp = Problem(prob, device=0, max_chains=1)
    H = mp.heights(torch.from_numpy(x).cuda())                     # device fp32 heights
    Hn = H.cpu().numpy().astype(np.float64)
    R = len(prob["ray_det"])

    def err(idx):
        p = sub(prob, idx)
        ll_d, G_d = Problem(p, device=0, max_chains=1).loglik_heights(H)
        o = oracle.Problem(p).loglik_grad_H(Hn)
        d = G_d.cpu().numpy().astype(np.float64)[0] - o["dldH"][0]
        return float(np.linalg.norm(d)), float(np.linalg.norm(o["dldH"][0])), float(ll_d.cpu().numpy()[0] - o["ll_dev"][0])

    full = err(np.arange(R))
    print(json.dumps({"chain": chain, "full_abs_err": full[0], "full_norm": full[1], "rel": full[0] / full[1]}), flush=True)
    thr = full[0] * 0.2
    stack = [np.arange(R)]
    found = []
    while stack:
        idx = stack.pop()
        e = err(idx)
        if e[0] < thr:
            continue
        if len(idx) <= 1:
            found.append((int(idx[0]), e))
            continue
        h = len(idx) // 2
        stack += [idx[:h], idx[h:]]
    for q, e in found:
        d = prob["ray_dir"][q]
        print(json.dumps({"ray": q, "abs_err": e[0], "ray_grad_norm": e[1], "dll": e[2],
                          "det": int(prob["ray_det"][q]), "dir": [float(v) for v in d]}), flush=True)


if __name__ == "__main__":
    main()
