#!/usr/bin/env python
"""Benchmark of the hot path: chain-sharded HMC on the Medium geometry.

One STEP = one HMC iteration over this rank's chains:
Philox momenta, L = 10 fused leapfrog steps (each = one log-posterior+gradient
evaluation over chains x rays: trace K2 + finish K3), Metropolis accept, the
a9 statistics (fixed-point acceptance sums, all-reduced over ranks for the
dual-averaging step size).  Metric = chain x ray log-posterior+gradient
evaluations per second, whole job: N * C * R * L * K / max-over-ranks time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mt|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...       (N > 1, one rank per GPU)

Workload = BASELINE configs[3] exactly: the Medium geometry and rays with
8,192 chains split evenly over the N GPUs (strong scaling: 8,192 chains on
one GPU at N = 1, 1,024 per GPU at N = 8).  --chains-total changes the total;
--weak keeps --chains-per-gpu fixed instead.  L2 is flushed (256 MiB write)
between timed steps, outside the event pairs.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "log-posterior+grad chain×ray evals/s"
UNIT = "chain×ray evals/s"
FP32_PEAK_NOMINAL = 148 * 128 * 2 * 1.965e9 / 1e12   # TFLOP/s: SMs x FP32 lanes x FMA x max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mt", choices=["mt", "reference"])
    ap.add_argument("--workload", default="chain_sharded",
                    choices=["chain_sharded", "ray_sharded", "tiny", "small", "medium"],
                    help="configs[3] (default, the headline), configs[4] (one chain, rays over the GPUs), or "
                         "configs[0..2] (tiny / small / medium: the config's own chain count per GPU)")
    ap.add_argument("--sampler", default="hmc", choices=["hmc", "nuts"],
                    help="fixed-L HMC (configs[3], default) or NUTS (SURVEY §8(f) f1; --max-depth)")
    ap.add_argument("--max-depth", type=int, default=8, help="NUTS: 2^max_depth leaves cap (P:662-669)")
    ap.add_argument("--model", default="exact", choices=["exact", "voxel"],
                    help="exact bilinear tracing (north_star) or the paper's voxel/linearised model (f3)")
    ap.add_argument("--states", default="posterior", choices=["posterior", "prior"],
                    help="near-posterior chain starts (headline) or prior draws (wide band: worst-case work, "
                         "SURVEY §8(d.1))")
    ap.add_argument("--nz", type=int, default=60, help="voxel model: layers (Δz = z_top/nz, reading R28)")
    ap.add_argument("--noncentred", action="store_true",
                    help="non-centred prior x = Q(r)^-1/2 z with sampled r (f2, P:570-584; implies --sample-r)")
    ap.add_argument("--sample-r", action="store_true",
                    help="hierarchical CAR r_l (SURVEY §8(f) f2): two more parameters per chain")
    ap.add_argument("--chains-total", type=int, default=8192)     # configs[3]
    ap.add_argument("--weak", action="store_true", help="fixed --chains-per-gpu per rank instead")
    ap.add_argument("--chains-per-gpu", type=int, default=1024)
    ap.add_argument("--leapfrog", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each timed HMC step from a CUDA graph (auto: HMC without a ray-shard communicator)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self, gpu_index=None):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            v = [t.strip() for t in line.split(",")]
            if len(v) < 9:
                continue
            if gpu_index is not None and v[0] != str(gpu_index):
                continue
            rows.append(v)
        os.unlink(self.f.name)
        post = False
        if not rows:   # a timed region shorter than one 200-ms sample: query once, right after it
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=20).stdout
                rows = [[t.strip() for t in ln.split(",")] for ln in out.splitlines()]
                rows = [v for v in rows if len(v) >= 9 and (gpu_index is None or v[0] == str(gpu_index))]
                post = True
            except Exception:
                rows = []
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip() == "Active"})
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        ck = {"sm_mhz": statistics.median(load) if load else None,
              "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}
        if post:
            ck["sampled"] = "once, right after the timed region (shorter than the 200-ms sampling period)"
        return ck


def cpu_baseline(seconds: float, chains: int = 4, name: str = "chain_sharded", nz: int = 0,
                 mode: str = "exact", states: str = "posterior"):
    """The fp64 oracle, as it stands, on this host's cores: the workload's
    geometry, `chains` chains x all its rays per evaluation, repeated for ~`seconds`.
    nz > 0: the voxel / linearised model's oracle (G rebuilt by every call, as the
    oracle does); mode "sample_r" / "noncentred": the f2 oracles; states "prior":
    prior-draw chain states."""
    import numpy as np

    import oracle
    from paper_2603_28907_b200 import inputs
    prob = inputs.make_problem(name)
    op = oracle.Problem(prob)
    cfg = inputs.CONFIGS[name]
    x = (inputs.prior_states(name, chains) if states == "prior"
         else inputs.chain_states(prob["x_true"], chains, cfg.seed)).astype(np.float64)
    rho = np.log(np.asarray(cfg.car_r) / (1.0 - np.asarray(cfg.car_r)))
    if mode == "sample_r":
        x = np.concatenate([x, np.broadcast_to(rho, (chains, 2))], axis=1)
    elif mode == "noncentred":
        from paper_2603_28907_b200.hmc import noncentred_state
        x = noncentred_state(x, rho, cfg.n, cfg.n).astype(np.float64)
    href = np.asarray(prob["H_true"], np.float32).astype(np.float64)
    t0 = time.perf_counter()
    n = 0
    while True:
        if nz:
            op.voxel_logpost_grad(x, href, nz)
        elif mode == "sample_r":
            op.logpost_grad_r(x)
        elif mode == "noncentred":
            op.logpost_grad_ncp(x)
        else:
            op.logpost_grad(x)
        n += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    what = (f" (voxel model, n_z={nz})" if nz else f" ({mode})" if mode != "exact" else "")
    return {"value": n * chains * op.R / dt, "unit": UNIT, "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"{name} geometry{what}, {chains} {'prior-draw' if states == 'prior' else 'near-posterior'} "
                      f"chain(s) x {op.R} rays per evaluation, "
                      f"{n} evaluations ({n * chains * op.R:.3g} chain-ray pairs) in {dt:.1f} s, fp64"}


def run_reference(args):
    """--impl reference: the oracle's HMC iteration (fp64 CPU) on a bounded sample."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_2603_28907_b200 import inputs
    cfg = inputs.CONFIGS["chain_sharded"]
    prob = inputs.make_problem("medium")
    op = oracle.Problem(prob)
    Cs = 2
    x = inputs.chain_states(prob["x_true"], Cs, cfg.seed, super_size=8).astype(np.float64)
    seed = inputs.philox_key(cfg)
    lg = lambda xx: (lambda o: (o["logp"], o["grad"]))(op.logpost_grad(xx))  # noqa: E731
    L = args.leapfrog
    for it in range(args.warmup):
        x, *_ = oracle.hmc_step(x, cfg.eps, L, lg, seed, it)
    times = []
    for it in range(args.steps):
        t0 = time.perf_counter()
        x, *_ = oracle.hmc_step(x, cfg.eps, L, lg, seed, args.warmup + it)
        times.append(time.perf_counter() - t0)
    T = sum(times)
    units = Cs * op.R * (L + 1) * args.steps   # L leapfrog evaluations + the initial one
    v = units / T
    lf_per_chain = L * args.steps / T          # leapfrog steps per second per chain (each chain: all rays)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic (seeded Medium geometry; counts = Poisson of the oracle's truth)",
            "config": {"workload": ("chain_sharded HMC iteration (BASELINE configs[3]: Medium geometry and rays, "
                                    f"{args.chains_total} chains over {args.gpus} GPU(s))"),
                       "global_chains": args.chains_total, "rays": op.R, "leapfrog_steps": L, "params": op.P,
                       "sample": f"{Cs} of the {args.chains_total} chains per timed HMC iteration (fp64 oracle)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"{Cs} chains x {op.R} rays x {L} leapfrog steps per HMC iteration"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "leapfrog_steps_per_s_per_chain": lf_per_chain}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    from paper_2603_28907_b200 import Problem, inputs
    from paper_2603_28907_b200.hmc import ChainShard

    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch N>1 with torchrun")
    # MT_BENCH_BACKEND=gloo (tests only): the N > 1 control flow with every rank on the
    # devices present (ranks may share one); the driver's multi-GPU runs use NCCL
    backend = os.environ.get("MT_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    dev = torch.device(f"cuda:{local}")

    ray = args.workload == "ray_sharded"
    cfg = inputs.CONFIGS[args.workload]
    dname = inputs.DATA_NAME[args.workload]
    prob = inputs.make_problem(args.workload)
    L = args.leapfrog
    tpath = os.path.join(ROOT, "data", "tuned_eps.json")
    tuned = json.load(open(tpath)).get(dname) if os.path.exists(tpath) else None
    eps = tuned["eps"] if tuned else cfg.eps   # sampling-phase ε from the warm-up (tools/tune_eps.py)
    if ray:
        # configs[4]: one chain, its 4,194,304 rays split over the ranks, in-library NCCL
        # all-reduce of [logp, grad] per evaluation; chains replicated on every rank
        from paper_2603_28907_b200.hmc import ray_sharded_problem
        C, offset = 1, 0
        x0 = inputs.chain_states(prob["x_true"], C, cfg.seed)
        # equal ray counts: the one-GPU shard table (profiles/r2_shard_balance.json) found them
        # within 5-8% of balanced, and cuts by band cells or by measured per-ray cost no better
        pb = ray_sharded_problem(prob, rank, ws, local, max_chains=C)
        R_total = len(prob["ray_det"])
        shard = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=L, eps0=eps, replicated=True)
    else:
        if args.workload in ("tiny", "small", "medium"):   # configs[0..2]: the config's chain count per GPU
            args.weak, args.chains_per_gpu = True, cfg.chains
        if args.weak:
            C = args.chains_per_gpu
        else:
            if args.chains_total % (8 * ws) or args.workload != "chain_sharded":
                raise SystemExit(f"--chains-total {args.chains_total} must split into super-chains of 8 per rank")
            C = args.chains_total // ws
        offset = rank * C
        x0 = inputs.chain_states(prob["x_true"], C, cfg.seed, chain_offset=offset,
                                 super_size=8 if args.workload == "chain_sharded" else 1)
        if args.states == "prior":
            x0 = np.ascontiguousarray(np.roll(inputs.prior_states(args.workload, C + offset), -offset, axis=0)[:C])
        rho = np.log(np.asarray(cfg.car_r) / (1.0 - np.asarray(cfg.car_r)))
        if args.noncentred:   # z = Q(r)^{1/2} x at the fixed-r value of ρ
            from paper_2603_28907_b200.hmc import noncentred_state
            x0 = noncentred_state(x0, rho, cfg.n, cfg.n)
        elif args.sample_r:   # ρ_l = logit(r_l) started at the fixed-r value
            x0 = np.concatenate([x0, np.broadcast_to(rho, (C, 2))], axis=1).astype(np.float32)
        pb = Problem(prob, device=local, max_chains=C, sample_r=args.sample_r, noncentred=args.noncentred)
        R_total = pb.R * ws   # (chain sharding: every rank traces all rays of its chains)
        shard = ChainShard(pb, x0, seed=inputs.philox_key(cfg), L=L, eps0=eps, chain_offset=offset,
                           n_chains_total=C * ws, sampler=args.sampler, max_depth=args.max_depth)
    voxel = args.model == "voxel"
    if voxel:   # R0 = R̂(H_ref), H_ref = the synthetic truth (stand-in for the expert model, R28)
        pb.voxel_model(args.nz, prob["H_true"])
        shard.refresh()
    R, P = pb.R, pb.P
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MiB > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    use_graph = args.graph == "on" or (args.graph == "auto" and args.sampler == "hmc" and not (ray and ws > 1))
    for w in range(args.warmup):   # (graph mode: the first warm-up step runs eagerly, then capture + replays)
        if use_graph and w > 0:
            shard.step_graph(sample=True, monitor=True)
        else:
            shard.step(adapt=False, sample=True, monitor=True)
    barrier()
    l2_peak = None
    if voxel:
        from paper_2603_28907_b200 import measure_l2_gather
        l2_peak = measure_l2_gather(local, 32 << 20)
        barrier()
    clocks = ClockSampler() if rank == 0 else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    pb.timing_start(args.steps * (L if args.sampler == "hmc" else 2 ** args.max_depth) + 8)
    d0 = pb.trace_counters()["deferred"]
    g0 = pb.voxel_gathered_bytes() if voxel else 0
    wall0 = time.perf_counter()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record()
        if use_graph:
            shard.step_graph(sample=True, monitor=True)
        else:
            shard.step(adapt=False, sample=True, monitor=True)
        ev[k][1].record()
    barrier()
    wall = time.perf_counter() - wall0
    ck = clocks.stop(gpu_index=None) if clocks else None
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    tm = pb.timing_read()
    cnt = pb.trace_counters()
    gathered = (pb.voxel_gathered_bytes() - g0) if voxel else 0
    if use_graph:
        # graph replays carry no host-side counters or per-launch events: the evaluations
        # are L per step, the launches those of one captured step, and the per-launch
        # kernel times come from one eager calibration step after the timed region
        evals_g = args.steps * L
        pb.timing_start(L + 8)
        shard.step(adapt=False, sample=True, monitor=True)
        torch.cuda.synchronize()
        cal, cal_cnt = pb.timing_read(), pb.trace_counters()
        per = 1.0 / max(cal["trace_launches"], 1)
        tm = {"trace_ms": cal["trace_ms"] * per * evals_g, "trace_launches": evals_g,
              "all_launches": shard.launches_per_graph_step * args.steps}
        cnt = {"deferred": cnt["deferred"], "defer_ms": cal_cnt["defer_ms"] * per * evals_g}
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    # evaluations of all chains x all rays (the trace launches: L per HMC step; one per
    # lockstep NUTS leaf, idle chains included)
    evals = tm["trace_launches"]
    units = (R_total * C if ray else ws * C * R) * evals
    value = units / (t_ms * 1e-3)

    # dominant kernel (K2 trace): algorithmic FP32 flops per launch / measured launch duration
    # (prior-draw states: the oracle's counts on prior draws, tools/count_work.py --prior)
    wc = json.load(open(os.path.join(ROOT, "data", "work_counts.json")))
    wkey = dname + "_prior" if args.states == "prior" and dname + "_prior" in wc else dname
    work = wc[wkey]
    F = work["flops_per_pair"]
    avg_trace_ms = tm["trace_ms"] / max(tm["trace_launches"], 1)       # K2 main + fp64 follow-up
    avg_defer_ms = cnt["defer_ms"] / max(tm["trace_launches"], 1)
    achieved = F * C * R / (avg_trace_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "trace_traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath)).get(args.workload + ("_prior" if args.states == "prior" else ""))
        traffic = tr.get("bytes_per_launch") if tr and tr.get("chains") == C else None
    from paper_2603_28907_b200 import measure_fp32_peak
    ffma_tf, ffma_mhz = measure_fp32_peak(local)
    roofline = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_NOMINAL, "unit": "TFLOP/s",
                "fp32_ffma_measured": ffma_tf, "fp32_ffma_measured_mhz": ffma_mhz,
                "frac": achieved / FP32_PEAK_NOMINAL, "traffic": traffic,
                "kernel": ("K2 = k_trace_rl (ray lanes)" if ray else "K2 = k_trace_cl (chain lanes)")
                          + " + k_trace_defer (fp64 follow-up), per launch pair",
                "flops_per_pair": F, "work_counts": f"data/work_counts.json[{wkey}]",
                "defer_share_of_trace": avg_defer_ms / avg_trace_ms,
                "deferred_pairs_per_launch": (cnt["deferred"] - d0) / max(tm["trace_launches"], 1),
                "trace_share_of_step": tm["trace_ms"] / t_ms if ws == 1 else None,
                "avg_trace_launch_ms": avg_trace_ms,
                "peak_note": "FP32 peak derived: 148 SMs x 128 lanes x 2 x 1.965 GHz (B200_PROFILING.md; "
                             "MEASURED_PEAKS.json has no FP32 entry); fp32_ffma_measured = mt_measure_fp32_peak "
                             "(independent FFMA chains, best of 10) on this device, for context; "
                             "F = algorithmic flops per chain x ray from the oracle's work counters with the "
                             "weights of SURVEY §8(d.3) (tools/count_work.py)"}

    if voxel:
        # V2 (λ̂ SpMV) + V3 (Gᵀ pass) are bound by L2-resident gathers of ΔR / r: 4 B per
        # chain and in-band G entry each (the V2 count, counted by the kernel; V3 gathers
        # the same entries), against the measured L2 gather bandwidth
        avg_vx_ms = tm["trace_ms"] / max(tm["trace_launches"], 1)
        ach = 2.0 * gathered / max(tm["trace_launches"], 1) / (avg_vx_ms * 1e-3) / 1e9
        vtraffic = None
        tpath = os.path.join(ROOT, "profiles", "voxel_traffic.json")
        if os.path.exists(tpath):
            tr = json.load(open(tpath)).get(args.workload + ("_prior" if args.states == "prior" else ""))
            vtraffic = tr.get("bytes_per_launch") if tr and tr.get("chains") == C else None
        info = pb.voxel_info()
        roofline = {"bound": "l2", "achieved": ach, "peak": l2_peak, "unit": "GB/s", "frac": ach / l2_peak,
                    "traffic": vtraffic,
                    "kernel": "V1 k_vx_rhat + V2 k_vx_fwd + V3 k_vx_bwd per evaluation (voxel model)",
                    "gathered_bytes_per_launch": 2.0 * gathered / max(tm["trace_launches"], 1),
                    "trace_share_of_step": tm["trace_ms"] / t_ms if ws == 1 else None,
                    "avg_eval_ms": avg_vx_ms, "nnz": info["nnz"], "n_grid": info["n_grid"],
                    "peak_note": "peak = mt_measure_l2_gather on this device (512-B rows at hashed indices of "
                                 "a 32 MiB L2-resident buffer, best of 10); achieved = algorithmic gather bytes "
                                 "(kernel-counted) / measured V1+V2+V3 time (DESIGN.md §7 voxel model)"}
        if C < 16:   # row lanes (one chain): the G stream (CSR + CSC, 8 B per entry each) from HBM binds
            hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
            gb = 16.0 * info["nnz"] / (avg_vx_ms * 1e-3) / 1e9
            roofline.update({"bound": "hbm", "achieved": gb, "peak": hbm, "frac": gb / hbm,
                             "peak_note": "peak = MEASURED_PEAKS.json hbm_gbs (copy bandwidth); achieved = G bytes "
                                          "(CSR + CSC, 16 B per non-zero; the in-band skip reads less) / "
                                          "measured V1+V2+V3 time (DESIGN.md §7 voxel model)"})

    e2e = None
    if not args.no_e2e:
        # the same metric through the public API with the chain state held in pinned host
        # memory: every step copies (x, logp, grad) host -> device, runs the step, and
        # copies (x, logp, grad, acceptance) device -> host
        xh = shard.x.cpu().pin_memory()
        gh = shard.grad.cpu().pin_memory()
        lph = shard.logp.cpu().pin_memory()
        aph = torch.empty(C, dtype=torch.float32).pin_memory()
        barrier()
        pb.timing_start(args.steps * (L if args.sampler == "hmc" else 2 ** args.max_depth) + 8)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(args.steps):
            shard.x.copy_(xh, non_blocking=True)
            shard.grad.copy_(gh, non_blocking=True)
            shard.logp.copy_(lph, non_blocking=True)
            if use_graph:
                shard.step_graph(sample=True, monitor=True)
            else:
                shard.step(adapt=False, sample=True, monitor=True)
            xh.copy_(shard.x, non_blocking=True)
            gh.copy_(shard.grad, non_blocking=True)
            lph.copy_(shard.logp, non_blocking=True)
            aph.copy_(shard.acc_prob, non_blocking=True)
        e1.record()
        barrier()
        evals_e2e = args.steps * L if use_graph else pb.timing_read()["trace_launches"]
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        units_e2e = (R_total * C if ray else ws * C * R) * evals_e2e
        state_bytes = C * (2 * P * 4 + 8)
        e2e = {"value": units_e2e / (float(te.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": state_bytes, "d2h_bytes_per_step": state_bytes + C * 4}

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    base = None
    if ws == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(args.cpu_seconds, chains=1 if ray else 4, name=args.workload,
                            nz=args.nz if voxel else 0,
                            mode="noncentred" if args.noncentred else "sample_r" if args.sample_r else "exact",
                            states=args.states)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic (seeded {'configs[4] 800 m' if ray else 'Medium'} geometry; counts = Poisson of the "
                    "oracle's truth; near-posterior chain states)",
            "config": {"workload": (f"ray_sharded HMC iteration (BASELINE configs[4]: one chain, {R_total} rays "
                                    f"over {ws} GPU(s))") if ray else
                                   ("chain_sharded HMC iteration (BASELINE configs[3]: Medium geometry and rays, "
                                    f"{C * ws} chains over {ws} GPU(s))") if args.workload == "chain_sharded" else
                                   (f"{args.workload} HMC iteration (BASELINE configs"
                                    f"[{['tiny', 'small', 'medium'].index(args.workload)}]: {C} chains per GPU, "
                                    f"{R} rays, {ws} GPU(s))"),
                       "chains_per_gpu": C, "global_chains": C if ray else C * ws, "rays": R_total if ray else R,
                       "rays_per_gpu": R, "params": P,
                       "leapfrog_steps": L, "parallelism": (f"ray-sharded x{ws}" if ray else f"chain-sharded x{ws}"),
                       "car_r": ("sampled, non-centred x = Q(r)^-1/2 z (f2)" if args.noncentred
                                 else "sampled (f2)" if args.sample_r else "fixed"),
                       "states": ("prior draws (wide band, worst-case work)" if args.states == "prior"
                                  else "near-posterior"),
                       "forward_model": (f"voxel/sigmoid/linearised (f3, P:242-390): n_z={args.nz}, gamma=1 m, "
                                         "R0 = R-hat(truth)") if voxel else "exact bilinear tracing (north_star)",
                       "phase": "sampling (fixed eps from the 100-iteration dual-averaging warm-up, "
                                "tools/tune_eps.py; Welford + all-reduced acceptance sums each step)",
                       "eps": eps,
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "launch": ("each step replayed from a CUDA graph (ChainShard.step_graph); per-launch kernel "
                                  "times from one eager step after the timed region") if use_graph else
                                 "eager launches"},
            "roofline": roofline, "cpu_baseline": base, "e2e": e2e, "clocks": ck,
            "gpu_launches": tm["all_launches"],
            "leapfrog_steps_per_s_per_chain": evals / (t_ms * 1e-3),
            "sampler": args.sampler if args.sampler == "hmc" else f"nuts (max_depth {args.max_depth})",
            "wall_s_timed_region": wall}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
