"""Locate a gradient parity failure: per-node ∂ℓ/∂H (device vs oracle on the
same fp32 heights), then per-ray device/oracle contributions to the worst node
(single-ray problems).  Test infrastructure.

  python tools/prior_debug.py <config> <chain> [--prior]
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


def main():
    name, c = sys.argv[1], int(sys.argv[2])
    prior = "--prior" in sys.argv
    cfg = inputs.CONFIGS[name]
    prob = inputs.make_problem(name)
    op = oracle.Problem(prob)
    x = (inputs.prior_states(name, cfg.chains) if prior else inputs.chain_states(prob["x_true"], cfg.chains, cfg.seed))
    mp = Problem(prob, device=0, max_chains=cfg.chains)
    H = mp.heights(torch.from_numpy(x).cuda())[c:c + 1].contiguous()
    ll_d, G_d = mp.loglik_heights(H)
    Hn = H.cpu().numpy().astype(np.float64)
    o = op.loglik_grad_H(Hn)
    Gd, Go = G_d.cpu().numpy()[0].astype(np.float64), o["dldH"][0]
    print(json.dumps({"ll_dev": float(ll_d[0]), "ll_ora": float(o["ll_dev"][0]),
                      "rel_l2_dldH": float(np.linalg.norm(Gd - Go) / np.linalg.norm(Go))}))
    diff = np.abs(Gd - Go).reshape(-1)
    top = np.argsort(-diff)[:5]
    for t in top:
        l, k = divmod(int(t), op.N)
        print(json.dumps({"surface": l, "node": divmod(k, op.ny), "dev": float(Gd.reshape(-1)[t]),
                          "ora": float(Go.reshape(-1)[t]), "absdiff": float(diff[t])}))
    l, k = divmod(int(top[0]), op.N)
    ni, nj = divmod(k, op.ny)
    # rays whose traversal touches a cell with corner (ni, nj)
    cand = []
    for q in range(op.R):
        ij, _, _ = op.traversal(q)
        if any(abs(int(i) - ni) <= 1 and abs(int(j) - nj) <= 1 and i <= ni <= i + 1 and j <= nj <= j + 1 for i, j in ij):
            cand.append(q)
    print("candidate rays", len(cand))
    rows = []
    for q in cand:
        sub = dict(prob)
        for key in ("ray_det", "ray_dir", "ray_w", "counts"):
            sub[key] = np.ascontiguousarray(prob[key][q:q + 1])
        m1 = Problem(sub, device=0, max_chains=1)
        _, g1 = m1.loglik_heights(H)
        o1 = oracle.Problem(sub).loglik_grad_H(Hn, with_sens=True)
        d = float(g1.cpu().numpy()[0].reshape(-1)[top[0]])
        r = float(o1["dldH"][0].reshape(-1)[top[0]])
        L, O, mg = oracle.Problem(sub).path_lengths(Hn, with_min_g1=True)
        rows.append((abs(d - r), q, d, r, float(mg[0, 0])))
    rows.sort(reverse=True)
    for e, q, d, r, mg in rows[:8]:
        print(json.dumps({"ray": q, "dev": d, "ora": r, "absdiff": e, "min_abs_g1": mg}))


if __name__ == "__main__":
    main()
