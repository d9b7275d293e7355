"""Chain sharding end to end on the GPU with two processes: two
ranks on the one available device, gloo for the host-side all-reduces (the
N-GPU bench uses NCCL for the same calls).  No kernel of one rank waits on the
other (chain sharding has no data-path collective), so sharing a device is
only a capacity stand-in.  Each rank runs ChainShard on its contiguous 32 of 64
global chains; the dual-averaging step size (from all-reduced fixed-point
acceptance sums) and every chain's final state must equal a single-process
64-chain run up to the summation order of the float atomics (one iteration:
dual averaging and HMC amplify such rounding chaotically over longer runs).
The R-hat all-reduce is covered with gloo on CPU (test_dist_cpu.py)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, out_dir, n_warm, n_samp):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_28907_b200 import Problem, inputs
    from paper_2603_28907_b200.hmc import ChainShard
    prob = inputs.make_problem("small")
    cfg = inputs.CONFIGS["small"]
    C_total = 64
    C = C_total // world
    off = rank * C
    x0 = inputs.chain_states(prob["x_true"], C, cfg.seed, chain_offset=off, super_size=8)
    pb = Problem(prob, device=0, max_chains=C)
    sh = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=10, eps0=cfg.eps, chain_offset=off,
                    n_chains_total=C_total)
    out = sh.run(n_warm, n_samp)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=sh.x.cpu().numpy(), eps=out["eps"],
             acc=np.array(out["warmup_accept"]), acc_prob=sh.acc_prob.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_chain_sharding_matches_one_process(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_2603_28907_b200 import Problem, inputs
    from paper_2603_28907_b200.hmc import ChainShard
    n_warm, n_samp = 1, 0   # one adapting iteration from the same ε: later ones amplify atomic-order rounding
    port = _free_port()
    mp.spawn(_run, args=(2, port, str(tmp_path), n_warm, n_samp), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"rank{k}.npz") for k in range(2))
    prob = inputs.make_problem("small")
    cfg = inputs.CONFIGS["small"]
    x0 = inputs.chain_states(prob["x_true"], 64, cfg.seed, super_size=8)
    pb = Problem(prob, device=0, max_chains=64)
    sh = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=10, eps0=cfg.eps)
    out = sh.run(n_warm, n_samp)
    # the all-reduced fixed-point acceptance gives both ranks the same global mean, hence
    # bit-identical dual-averaging step sizes; the single run agrees up to rounding
    assert float(r0["eps"]) == float(r1["eps"]) and np.array_equal(r0["acc"], r1["acc"])
    assert np.allclose(r0["acc"], np.array(out["warmup_accept"]), rtol=1e-3)
    assert float(r0["eps"]) == pytest.approx(out["eps"], rel=1e-3)
    # every chain (global id) made the same HMC move as in the single process
    ap = np.concatenate([r0["acc_prob"], r1["acc_prob"]])
    assert np.allclose(ap, sh.acc_prob.cpu().numpy(), atol=1e-3)
    x_sh = np.concatenate([r0["x"], r1["x"]])
    x_one = sh.x.cpu().numpy()
    rel = np.linalg.norm(x_sh - x_one, axis=1) / np.linalg.norm(x_one, axis=1)
    assert np.mean(rel < 1e-5) > 0.95, rel     # (rounding can flip an accept sitting on its threshold)
