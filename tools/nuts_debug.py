"""GPU NUTS vs oracle NUTS, chain by chain, with the oracle's decision margins
(log u minus threshold) and which oracle leaf the GPU's result equals.
Debugging aid; test infrastructure (imports oracle/)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs  # noqa: E402


def main():
    name, C, md = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    cfg = inputs.CONFIGS[name]
    prob = inputs.make_problem(name)
    op = oracle.Problem(prob)
    mp = Problem(prob, device=0, max_chains=C)
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
    import json
    e = json.load(open(os.path.join(ROOT, "data", "tuned_eps.json"))).get(name, {}).get("eps", cfg.eps) * 2
    seed, it = inputs.philox_key(cfg), 11
    x = torch.from_numpy(x0).cuda()
    logp, grad = mp.logpost_grad(x)
    lp_dev0 = logp.cpu().numpy().copy()
    eps = torch.full((C,), e, dtype=torch.float32, device="cuda")
    acc, depth, nl = mp.nuts_step(x, logp, grad, eps, md, seed, it)
    xd = x.cpu().numpy().astype(np.float64)
    lg1 = lambda th: (lambda o: (o["logp"][0], o["grad"][0]))(op.logpost_grad(th[None]))  # noqa: E731
    for c in range(C):
        lp0, g0 = lg1(x0[c].astype(np.float64))
        tr = []
        ref = oracle.nuts_step(x0[c], lp0, g0, e, lg1, seed, it, c, max_depth=md, trace=tr)
        err = np.linalg.norm(xd[c] - ref["x"]) / np.linalg.norm(ref["x"])
        near = min(abs(m) for _, m, _ in tr)
        match = [k for k, (_, _, th) in enumerate(tr) if np.linalg.norm(xd[c] - th) / np.linalg.norm(th) < 1e-3]
        print(f"chain {c}: dev depth {depth[c].item()} leaves {nl[c].item()} | ora depth {ref['depth']} leaves "
              f"{ref['n_leaves']} | x err {err:.2e} | closest margin {near:.2e} | dev x = oracle choice #{match} "
              f"| lp0 dev {lp_dev0[c]:.6f} ora {lp0:.6f}")
        # the same algorithm (oracle code) driven by the CUDA log-posterior
        mp1 = Problem(prob, device=0, max_chains=1)

        def lg1_gpu(th):
            lp_, g_ = mp1.logpost_grad(torch.from_numpy(np.asarray(th, np.float32)[None]).cuda())
            return float(lp_.cpu()[0]), g_.cpu().numpy()[0].astype(np.float64)
        lpg, gg = lg1_gpu(x0[c])
        trg = []
        refg = oracle.nuts_step(x0[c].astype(np.float64), lpg, gg, e, lg1_gpu, seed, it, c, max_depth=md, trace=trg)
        errg = np.linalg.norm(xd[c] - refg["x"]) / np.linalg.norm(refg["x"])
        print(f"   oracle-NUTS on CUDA evaluations: depth {refg['depth']} leaves {refg['n_leaves']} x err vs kernel NUTS {errg:.2e}")
        for k, ((kind, m, th), (_, mg, thg)) in enumerate(zip(tr, trg)):
            dx = np.linalg.norm(th - thg) / np.linalg.norm(th)
            print(f"     {k:3d} {kind:5s} margin {m:+.4e} cuda-eval margin {mg:+.4e} |Δθ| {dx:.1e} {'TAKE' if m < 0 else ''}")


if __name__ == "__main__":
    main()
