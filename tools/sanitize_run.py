"""Small end-to-end run of every libmt entry point family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run): tiny and
small problems, both trace kernels (chain lanes, ray lanes), the deferred-pair
kernel, path lengths, HMC with statistics, a one-rank NCCL communicator.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_28907_b200 import Problem, comm_unique_id, inputs  # noqa: E402
from paper_2603_28907_b200.hmc import ChainShard  # noqa: E402


def main():
    for name, C in (("tiny", 4), ("small", 64), ("small", 3)):
        prob = inputs.make_problem(name)
        cfg = inputs.CONFIGS[name]
        pb = Problem(prob, device=0, max_chains=C)
        x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
        x = torch.from_numpy(x0).cuda()
        lp, g = pb.logpost_grad(x)
        H = torch.from_numpy(inputs.perturbed_heights(prob["H_true"], C, 5)).cuda()
        pb.path_lengths(H)
        pb.loglik_heights(H)
        sh = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=3, eps0=cfg.eps)
        sh.run(2, 3)
        print(name, C, "logp", float(lp[0]), "deferred", pb.trace_counters()["deferred"])
    pb = Problem(inputs.make_problem("tiny"), device=0, max_chains=4)
    pb.attach_comm(comm_unique_id(), 0, 1)
    x = torch.from_numpy(inputs.chain_states(inputs.make_problem("tiny")["x_true"], 4, 1)).cuda()
    pb.logpost_grad(x)
    pb.detach_comm()
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
