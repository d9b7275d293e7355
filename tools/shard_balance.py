"""One-GPU simulated ray-shard table (configs[4]): for k = 2, 4, 8 ray
shards (equal ray counts vs cut by trace work, hmc.ray_shards_weighted), build each
shard's problem on this one device and time its evaluation (trace + K3; the
all-reduce is not part of a shard's own time); print per-shard times and max/mean.

  python tools/shard_balance.py [--reps 20] > gpurun_out/shard_balance.json
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
from paper_2603_28907_b200.hmc import balanced_ray_shards, ray_shards  # noqa: E402


def time_shard(prob, lo, hi, x, reps):
    pb = Problem(prob, device=0, max_chains=1, ray_lo=lo, ray_hi=hi)
    lp, g = pb.logpost_grad(x)
    for _ in range(3):
        pb.logpost_grad(x, lp, g)
    torch.cuda.synchronize()
    pb.timing_start(reps + 4)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pb.logpost_grad(x, lp, g)
    e1.record()
    torch.cuda.synchronize()
    tm = pb.timing_read()
    return e0.elapsed_time(e1) / reps, tm["trace_ms"] / tm["trace_launches"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    prob = inputs.make_problem("ray_sharded")
    cfg = inputs.CONFIGS["ray_sharded"]
    x0 = inputs.chain_states(prob["x_true"], 1, cfg.seed)
    x = torch.from_numpy(x0).cuda()
    R = len(prob["ray_det"])
    out = {"config": "ray_sharded (configs[4]): 1 chain, %d rays; per-shard evaluation time on ONE B200" % R}
    for k in (2, 4, 8):
        for how, sh in (("equal_rays", ray_shards(R, k)),
                        ("band_cells", balanced_ray_shards(prob, x0[0], k, 0, measured=False)),
                        ("measured_cost", balanced_ray_shards(prob, x0[0], k, 0))):
            ts = [time_shard(prob, lo, hi, x, a.reps) for lo, hi in sh]
            ev = [t[0] for t in ts]
            tr = [t[1] for t in ts]
            out[f"k{k}_{how}"] = {"ranges": sh, "eval_ms": ev, "trace_ms": tr,
                                  "eval_max_over_mean": max(ev) / (sum(ev) / k),
                                  "trace_max_over_mean": max(tr) / (sum(tr) / k)}
            print(f"k={k} {how}: eval max/mean {max(ev) / (sum(ev) / k):.3f}, trace max/mean "
                  f"{max(tr) / (sum(tr) / k):.3f}", file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
