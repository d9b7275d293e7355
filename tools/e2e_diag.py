"""End-to-end gradient diagnosis: device ∇ₓ vs the
oracle from fp64 heights, and vs the oracle fed the fp32-rounded heights
(the "heights are fp32 quantities" convention), to separate kernel error
from the conditioning of fp32 height rounding (HP2).  Test infrastructure.

  python tools/e2e_diag.py <config> [chain ...] [--prior]   (--prior: prior-draw states)
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


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    name = sys.argv[1]
    prior = "--prior" in sys.argv
    chains = [int(c) for c in sys.argv[2:] if c != "--prior"] or [0]
    cfg = inputs.CONFIGS[name]
    prob = inputs.make_problem(name)
    op = oracle.Problem(prob)
    mp = Problem(prob, device=0, max_chains=cfg.chains)
    x = (inputs.prior_states(name, cfg.chains) if prior
         else inputs.chain_states(prob["x_true"], cfg.chains, cfg.seed))
    lp, g = mp.logpost_grad(torch.from_numpy(x).cuda())
    g = g.cpu().numpy().astype(np.float64)
    ref = op.logpost_grad(x[chains].astype(np.float64))
    for k, c in enumerate(chains):
        xc = x[c].astype(np.float64)
        H, dH = op.heights(xc)
        H32 = H.astype(np.float32).astype(np.float64)
        o32 = op.loglik_grad_H(H32[None], with_sens=True)
        G = o32["dldH"][0]
        gx = np.stack([G[0] * dH[0] + G[1] * dH[1], G[1] * dH[2]]).reshape(-1)
        n = op.nx
        for l in range(2):
            _, gp = oracle.prior_surface(xc.reshape(2, -1)[l].reshape(n, -1), op.prob["car_r"][l]) \
                if False else (None, None)
        # prior gradient: difference oracle(fp64 H) grad minus its likelihood part
        o64 = op.loglik_grad_H(H[None], with_sens=True)
        G64 = o64["dldH"][0]
        gx64 = np.stack([G64[0] * dH[0] + G64[1] * dH[1], G64[1] * dH[2]]).reshape(-1)
        prior_g = ref["grad"][k] - gx64
        g32 = gx + prior_g
        print(json.dumps({"config": name, "chain": c,
                          "dev_vs_ora64": rel(g[c], ref["grad"][k]),
                          "dev_vs_ora_fp32H": rel(g[c], g32),
                          "ora_fp32H_vs_ora64": rel(g32, ref["grad"][k]),
                          "sens64": float(o64["sens"][0]), "sens32": float(o32["sens"][0]),
                          "max_abs_diff_node": int(np.argmax(np.abs(g[c] - ref["grad"][k]))),
                          "grad_norm": float(np.linalg.norm(ref["grad"][k]))}), flush=True)


if __name__ == "__main__":
    main()
