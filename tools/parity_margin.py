"""Parity MARGINS (error / tolerance, worst case) of the CUDA path against the
oracle: the quantities the -m gpu tests bound, printed instead of asserted, so
that a kernel change can be judged by how close it comes to the tolerances.
Test infrastructure (imports oracle/).  MT_LIB selects a library variant.

  python tools/parity_margin.py [configs...]
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

PLAN = {"tiny": (4, 4, None), "small": (8, 8, None), "medium": (2, 2, [0, 511, 1023]),
        "ray_sharded": (1, 1, [0])}


def main():
    names = sys.argv[1:] or ["tiny", "small", "medium"]
    for name in names:
        Cp, Cl, e2e = PLAN[name]
        cfg = inputs.CONFIGS[name]
        prob = inputs.make_problem(name)
        op = oracle.Problem(prob)
        C = cfg.chains
        mp = Problem(prob, device=0, max_chains=C)
        out = {"config": name, "lib": os.environ.get("MT_LIB", "default")}
        H = inputs.perturbed_heights(prob["H_true"], Cp, 100 + Cp, scale=2.0)
        L_d, O_d = mp.path_lengths(torch.from_numpy(H).cuda())
        L_o, O_o = op.path_lengths(H.astype(np.float64))
        err = np.abs(L_d.cpu().numpy().astype(np.float64) - L_o).max(2) / (1e-5 * L_o.sum(2))
        out["path_len_margin_max"] = float(err.max())
        out["path_len_pairs_over_0.5"] = int((err > 0.5).sum())
        H = inputs.perturbed_heights(prob["H_true"], Cl, 200 + Cl, scale=1.0)
        ll_d, G_d = mp.loglik_heights(torch.from_numpy(H).cuda())
        ref = op.loglik_grad_H(H.astype(np.float64))
        out["ll_margin_max"] = float(np.max(np.abs(ll_d.cpu().numpy() - ref["ll_dev"]) / (1e-4 * np.abs(ref["ll_dev"]))))
        G = G_d.cpu().numpy().astype(np.float64)
        out["dldH_margin_max"] = float(max(np.linalg.norm(G[c] - ref["dldH"][c]) / (1e-3 * np.linalg.norm(ref["dldH"][c]))
                                           for c in range(Cl)))
        x = inputs.chain_states(prob["x_true"], C, cfg.seed)
        lp, g = mp.logpost_grad(torch.from_numpy(x).cuda())
        chains = np.arange(C) if e2e is None else np.array(e2e)
        ro = op.logpost_grad(x[chains].astype(np.float64))
        lp, g = lp.cpu().numpy(), g.cpu().numpy().astype(np.float64)
        out["e2e_logp_margin_max"] = float(max(abs(lp[c] - ro["logp"][k]) / (1e-4 * abs(ro["logp"][k])) for k, c in enumerate(chains)))
        out["e2e_grad_margin_max"] = float(max(np.linalg.norm(g[c] - ro["grad"][k]) / (1e-3 * np.linalg.norm(ro["grad"][k]))
                                               for k, c in enumerate(chains)))
        out["deferred_total"] = mp.trace_counters()["deferred"]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
