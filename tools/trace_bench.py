"""Time mt_logpost_grad alone (K1 + K2 + K3) on a config, for kernel tuning.

  python tools/trace_bench.py [config] [--chains C] [--reps N]
Env MT_TRACE_K / MT_TRACE_S override the trace launch shape.
Prints chain x ray evals/s, the trace kernel's share and its algorithmic TFLOP/s.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_28907_b200 import Problem, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="medium")
    ap.add_argument("--chains", type=int, default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ncp", action="store_true", help="non-centred parameterisation (f2)")
    ap.add_argument("--prior", action="store_true", help="prior-draw chain states (worst-case band)")
    ap.add_argument("--voxel", type=int, default=0, help="n_z > 0: time the f3 voxel / linearised model")
    a = ap.parse_args()
    cfg = inputs.CONFIGS[a.config]
    C = a.chains or cfg.chains
    prob = inputs.make_problem(a.config)
    pb = Problem(prob, device=0, max_chains=C, noncentred=a.ncp)
    if a.voxel:
        import time
        t0 = time.time()
        pb.voxel_model(a.voxel, prob["H_true"])
        print("voxel setup", pb.voxel_info(), f"{time.time() - t0:.2f} s", flush=True)
    x = torch.from_numpy(inputs.prior_states(a.config, C) if a.prior
                         else inputs.chain_states(prob["x_true"], C, cfg.seed)).cuda()
    if a.ncp:
        from paper_2603_28907_b200.hmc import noncentred_state
        rho = np.log(np.asarray(cfg.car_r) / (1 - np.asarray(cfg.car_r)))
        x = torch.from_numpy(noncentred_state(x.cpu().numpy(), rho, cfg.n, cfg.n)).cuda()
    lp, g = pb.logpost_grad(x)
    for _ in range(3):
        pb.logpost_grad(x, lp, g)
    torch.cuda.synchronize()
    pb.timing_start(a.reps + 4)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        pb.logpost_grad(x, lp, g)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    tm = pb.timing_read()
    cnt = pb.trace_counters()
    tr = tm["trace_ms"] / tm["trace_launches"]
    wall = json.load(open(os.path.join(ROOT, "data", "work_counts.json")))
    key = inputs.DATA_NAME[a.config]
    work = wall.get(key + "_prior", wall[key]) if a.prior else wall[key]
    F = work["flops_per_pair"]
    pairs = C * pb.R
    print(json.dumps({"config": a.config, "ncp": a.ncp, "states": "prior" if a.prior else "near-posterior", "C": C, "R": pb.R, "K": os.environ.get("MT_TRACE_K", "auto"),
                      "S": os.environ.get("MT_TRACE_S", "auto"), "ms_per_eval": ms, "trace_ms": tr,
                      "trace_share": tr / ms, "defer_ms": cnt["defer_ms"] / a.reps,
                      "deferred_per_eval": cnt["deferred"] / (a.reps + 4), "lib": os.environ.get("MT_LIB", "default"), "evals_per_s": pairs / (ms * 1e-3),
                      "trace_alg_tflops": F * pairs / (tr * 1e-3) / 1e12}))


if __name__ == "__main__":
    main()
