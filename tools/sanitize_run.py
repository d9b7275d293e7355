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
    # widenings: voxel model (chain and row lanes), non-centred (clusters), mass, NUTS,
    # prior-draw states (second walk, queue), summaries
    prob = inputs.make_problem("small")
    cfg = inputs.CONFIGS["small"]
    for C in (40, 3):
        pb = Problem(prob, device=0, max_chains=C)
        x = torch.from_numpy(inputs.chain_states(prob["x_true"], C, cfg.seed)).cuda()
        pb.voxel_model(20, prob["H_true"])
        lp, g = pb.logpost_grad(x)
        pb.voxel_model(0)
        pb.set_inverse_mass(torch.full((pb.P,), 0.7, device="cuda"))
        lp, g = pb.logpost_grad(x)
        eps = torch.full((C,), 1e-5, device="cuda")
        pb.hmc_step(x, lp, g, eps, 3, 5, 0)
        pb.nuts_step(x, lp, g, eps, 3, 5, 1)
        acc, mx, ml = pb.summary_buffers(20)
        pb.summary_update(x, lp, acc, 20, 10.0, mx, ml)
        xp = torch.from_numpy(inputs.prior_states("small", C)).cuda()
        pb.logpost_grad(xp)
        print("widenings", C, float(lp[0]))
    from paper_2603_28907_b200.hmc import noncentred_state
    for C in (2, 20):
        pb = Problem(prob, device=0, max_chains=C, noncentred=True)
        v = torch.from_numpy(noncentred_state(inputs.chain_states(prob["x_true"], C, cfg.seed), (2.5, 2.0),
                                              cfg.n, cfg.n)).cuda()
        lp, g = pb.logpost_grad(v)
        pb.hmc_step(v, lp, g, torch.full((C,), 1e-4, device="cuda"), 3, 5, 0)
        print("noncentred", C, float(lp[0]))
    pb = Problem(inputs.make_problem("tiny"), device=0, max_chains=4)
    pb.attach_comm(comm_unique_id(), 0, 1)
    x = torch.from_numpy(inputs.chain_states(inputs.make_problem("tiny")["x_true"], 4, 1)).cuda()
    pb.logpost_grad(x)
    pb.detach_comm()
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
