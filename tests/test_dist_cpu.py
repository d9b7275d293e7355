"""Multi-process host logic of chain sharding, on CPU with gloo (world_size 2).

What the N-GPU bench relies on, checked without GPUs:
  * the global chain ids a rank owns give exactly the chain states of the
    unsharded run (Philox streams and initial states keyed by global id);
  * the fixed-point acceptance sums all-reduced over ranks give the SAME mean
    acceptance, hence the same dual-averaging step size, on every rank and as
    an unsharded run (order-independent integer sums, HP9);
  * R-hat partial sums all-reduced over ranks equal the single-process R-hat
    computed from all chains at once;
  * ray sharding (configs[4] logic): hmc.ray_shards partitions the rays, each
    rank's partial log-posterior/gradient (likelihood of its shard, prior on
    shard 0 only — here computed by the oracle, test infrastructure) summed by
    all_reduce equals the unsharded result, identically on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_28907_b200 import inputs
from paper_2603_28907_b200.hmc import (DualAveraging, nested_rhat_from_partials, ray_shards, ray_shards_weighted,
                                       rhat_from_partials)

WS = 2
C_PER = 8
P = 16


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fixed_point(acc):
    """Host mirror of k_accept_sum: Σ round(a·2^32) and the count, int64."""
    return np.array([np.sum(np.rint(np.asarray(acc, np.float64) * 4294967296.0).astype(np.int64)),
                     len(acc)], np.int64)


def welford(xs):
    n = len(xs)
    mean = np.zeros_like(xs[0])
    m2 = np.zeros_like(xs[0])
    for k, x in enumerate(xs, 1):
        d = x - mean
        mean = mean + d / k
        m2 = m2 + d * (x - mean)
    return mean, m2, n


def make_draws(n_iter, n_chains):
    rng = np.random.default_rng(123)
    return rng.standard_normal((n_iter, n_chains, P)) * 0.7 + rng.standard_normal((1, n_chains, P)) * 0.2


def shard_problem(prob, lo, hi):
    keys = ("ray_det", "ray_dir", "ray_w", "counts")
    return dict(prob, **{k: np.asarray(prob[k])[lo:hi] for k in keys})


def ray_shard_partial_sum(rank):
    import oracle
    prob = inputs.make_problem("tiny")
    x = inputs.chain_states(prob["x_true"], 2, inputs.CONFIGS["tiny"].seed).astype(np.float64)
    lo, hi = ray_shards(len(prob["ray_det"]), WS)[rank]
    o = oracle.Problem(shard_problem(prob, lo, hi)).logpost_grad(x)
    logp = o["logp"] - (0.0 if rank == 0 else o["prior"])      # prior on shard 0 only
    grad = o["grad"].copy()
    if rank != 0:                                               # remove the prior gradient
        n = int(np.sqrt(x.shape[1] // 2))
        for c in range(2):
            for l in range(2):
                _, gp = oracle.prior_surface(x[c].reshape(2, n, n)[l], prob["car_r"][l])
                grad[c].reshape(2, n, n)[l] -= gp
    t = torch.from_numpy(np.concatenate([logp, grad.ravel()]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.numpy()


def worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        res = {}
        # 1. chain partition
        cfg = inputs.CONFIGS["small"]
        xt = inputs.make_problem("small")["x_true"]
        res["x0"] = inputs.chain_states(xt, C_PER, cfg.seed, chain_offset=rank * C_PER, super_size=8)
        # 2. dual averaging driven by all-reduced fixed-point acceptance sums
        rng = np.random.default_rng(7)
        acc_all = rng.uniform(0, 1, size=(20, WS * C_PER))
        da = DualAveraging(1e-3)
        eps = []
        for it in range(20):
            t = torch.from_numpy(fixed_point(acc_all[it, rank * C_PER:(rank + 1) * C_PER]))
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            s, n = (int(v) for v in t.tolist())
            eps.append(da.update(s / 4294967296.0 / n))
        res["eps"] = eps
        # 3. R-hat partials
        draws = make_draws(30, WS * C_PER)[:, rank * C_PER:(rank + 1) * C_PER]
        mean, m2, n = welford(list(draws))
        part = np.stack([mean.sum(0), (mean ** 2).sum(0), (m2 / (n - 1)).sum(0)])
        t = torch.from_numpy(part)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        res["rhat"] = rhat_from_partials(t.numpy(), WS * C_PER, n)
        # 3b. nested R-hat partials (super-chains of 8 never straddle ranks)
        from test_nested_rhat import partials_numpy
        part_n, Kr = partials_numpy(draws, 8)
        t = torch.from_numpy(part_n)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        res["nested"] = nested_rhat_from_partials(t.numpy(), WS * C_PER // 8)
        # 4. ray sharding: partial [logp, grad] of this rank's ray shard, all-reduced
        res["ray"] = ray_shard_partial_sum(rank)
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, port, out)) for r in range(WS)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    return dict(out)


def test_chain_partition_matches_unsharded(results):
    cfg = inputs.CONFIGS["small"]
    xt = inputs.make_problem("small")["x_true"]
    whole = inputs.chain_states(xt, WS * C_PER, cfg.seed, super_size=8)
    got = np.concatenate([results[r]["x0"] for r in range(WS)])
    assert np.array_equal(got, whole)


def test_step_size_identical_on_all_ranks_and_unsharded(results):
    assert results[0]["eps"] == results[1]["eps"]
    rng = np.random.default_rng(7)
    acc_all = rng.uniform(0, 1, size=(20, WS * C_PER))
    da = DualAveraging(1e-3)
    ref = []
    for it in range(20):
        s, n = fixed_point(acc_all[it])
        ref.append(da.update(int(s) / 4294967296.0 / int(n)))
    assert results[0]["eps"] == ref          # bit-identical: integer sums are order-free


def test_rhat_from_allreduced_partials(results):
    draws = make_draws(30, WS * C_PER)            # [iter][chain][param]
    n, m = draws.shape[0], draws.shape[1]
    cm = draws.mean(0)
    B = n * cm.var(0, ddof=1)
    W = draws.var(0, ddof=1).mean(0)
    ref = np.sqrt(((n - 1) / n * W + B / n) / W)  # Gelman-Rubin (P:684-687 cites the nested form)
    assert np.allclose(results[0]["rhat"], ref, rtol=1e-10)
    assert np.allclose(results[1]["rhat"], ref, rtol=1e-10)


def test_ray_sharded_partials_sum_to_unsharded(results):
    import oracle
    prob = inputs.make_problem("tiny")
    x = inputs.chain_states(prob["x_true"], 2, inputs.CONFIGS["tiny"].seed).astype(np.float64)
    ref = oracle.Problem(prob).logpost_grad(x)
    want = np.concatenate([ref["logp"], ref["grad"].ravel()])
    assert np.array_equal(results[0]["ray"], results[1]["ray"])      # identical on every rank
    assert np.allclose(results[0]["ray"], want, rtol=1e-10, atol=1e-8)


def test_nested_rhat_from_allreduced_partials(results):
    from test_nested_rhat import nested_rhat_direct
    draws = make_draws(30, WS * C_PER)
    want = nested_rhat_direct(draws, 8)
    for r in range(WS):
        assert np.allclose(results[r]["nested"], want, rtol=1e-10)


def test_weighted_ray_shards_balance_the_work():
    """ray_shards_weighted: contiguous, covering, non-empty ranges whose work
    (band cells + per-ray cost) differs from the mean by at most one ray's work."""
    rng = np.random.default_rng(5)
    work = rng.integers(0, 30, 4096)
    work[:1024] = 0                      # e.g. an edge detector's rays that leave below the band
    for world in (1, 2, 4, 8):
        sh = ray_shards_weighted(work, world)
        assert sh[0][0] == 0 and sh[-1][1] == len(work)
        assert all(a < b for a, b in sh) and all(sh[k][1] == sh[k + 1][0] for k in range(world - 1))
        tot = np.array([np.sum(work[a:b] + 2.0) for a, b in sh])
        assert np.all(np.abs(tot - tot.mean()) <= work.max() + 2.0), tot
    eq = ray_shards(len(work), 4)
    tot_eq = np.array([np.sum(work[a:b] + 2.0) for a, b in eq])
    assert tot_eq.max() / tot_eq.mean() > 1.2     # equal counts are badly balanced here
