"""HMC driver over the C ABI: one chain shard per process/GPU.

Host-side logic only (scalars): step-size adaptation by dual averaging
(Hoffman & Gelman 2014, Alg. 5 — the "robust adaptation procedure" of
P:652-653, reading R20) on ONE global log ε driven by the all-chain mean
acceptance probability, and the R-hat assembly from per-rank partial sums
(reading R21).  All per-chain work (momenta, leapfrog, Metropolis,
acceptance sums, Welford) runs in libmt kernels.

Chain sharding: chains are split contiguously over ranks,
Philox streams are keyed by the GLOBAL chain id and acceptance sums are exact
int64 fixed-point, so every rank computes the same ε and per-chain results do
not depend on the number of GPUs.  The only collectives are an all-reduce of
two int64 per warm-up iteration and of 3P doubles for R-hat at the end.

Ray sharding (BASELINE configs[4]): the rays are split into contiguous ranges,
one per rank (ray_shards); every rank holds the same chains (replicated) and
its problem computes the shard's partial log-likelihood and gradient; the
library's in-stream NCCL all-reduce (Problem.attach_comm, include/mt.h) sums
them before every kick, so all ranks follow identical trajectories and no
sampler statistic needs a cross-rank reduction (ChainShard(replicated=True)).
"""
from __future__ import annotations

import contextlib
import math
from typing import Optional

import numpy as np


def noncentred_state(x: np.ndarray, rho, nx: int, ny: int) -> np.ndarray:
    """Host helper: the non-centred state (z_0, z_1, ρ_0, ρ_1) with U(r_l) z_l = x_l, i.e.
    z_l = Q(r_l)^{1/2} x_l (numpy 2-D FFT on the torus), for starting non-centred chains
    (Problem(noncentred=True)) from centred states x [C][2N].  Not on the hot path."""
    x = np.asarray(x, np.float64)
    C, N = x.shape[0], nx * ny
    a = np.arange(nx)[:, None]
    b = np.arange(ny)[None, :]
    cab = 2.0 * (np.cos(2 * np.pi * a / nx) + np.cos(2 * np.pi * b / ny))
    out = np.zeros((C, 2 * N + 2), np.float64)
    for l in range(2):
        r = 1.0 / (1.0 + np.exp(-float(rho[l])))
        xl = x[:, l * N:(l + 1) * N].reshape(C, nx, ny)
        zl = np.real(np.fft.ifft2(np.fft.fft2(xl) * np.sqrt(4.0 - r * cab)))
        out[:, l * N:(l + 1) * N] = zl.reshape(C, N)
        out[:, 2 * N + l] = rho[l]
    return out.astype(np.float32)


class DualAveraging:
    """Nesterov dual averaging of log ε towards a target acceptance δ."""

    def __init__(self, eps0: float, target: float = 0.8, gamma: float = 0.05, t0: float = 10.0,
                 kappa: float = 0.75):
        self.mu = math.log(10.0 * eps0)
        self.target, self.gamma, self.t0, self.kappa = target, gamma, t0, kappa
        self.m = 0
        self.hbar = 0.0
        self.log_eps = math.log(eps0)
        self.log_eps_bar = 0.0

    def update(self, alpha: float) -> float:
        self.m += 1
        m = self.m
        w = 1.0 / (m + self.t0)
        self.hbar = (1.0 - w) * self.hbar + w * (self.target - alpha)
        self.log_eps = self.mu - math.sqrt(m) / self.gamma * self.hbar
        mk = m ** (-self.kappa)
        self.log_eps_bar = mk * self.log_eps + (1.0 - mk) * self.log_eps_bar
        return math.exp(self.log_eps)

    def final(self) -> float:
        """The averaged step size; with no update yet, the current one (ε₀)."""
        return math.exp(self.log_eps_bar if self.m > 0 else self.log_eps)


def mass_windows(n_warmup: int, init: int = 75, term: int = 50, base: int = 25):
    """Stan-style slow-adaptation windows [(start, end)] of the warm-up (R19b):
    an initial buffer, doubling windows, a terminal buffer; scaled 15% / 75% / 10%
    when the warm-up is shorter than init + term + base.  Empty below 20 iterations."""
    if n_warmup < 20:
        return []
    if init + term + base > n_warmup:
        init, term = int(0.15 * n_warmup), int(0.1 * n_warmup)
        base = n_warmup - init - term
    out, start, w = [], init, base
    end_slow = n_warmup - term
    while start < end_slow:
        end = start + w
        if end + 2 * w > end_slow:       # the last window absorbs the remainder
            end = end_slow
        out.append((start, end))
        start, w = end, 2 * w
    return out


def rhat_from_partials(part: np.ndarray, n_chains: int, n: int) -> np.ndarray:
    """Classic R-hat per parameter from Σ m̄_c, Σ m̄_c², Σ s²_c over all chains."""
    s1, s2, sv = part
    mean = s1 / n_chains
    B_over_n = (s2 - n_chains * mean ** 2) / (n_chains - 1)   # variance of chain means
    W = sv / n_chains
    var_plus = (n - 1) / n * W + B_over_n
    return np.sqrt(var_plus / W)


def ray_shards(R: int, world: int):
    """Contiguous ray ranges [lo, hi) of the caller's ray order, one per rank,
    sizes differing by at most one."""
    if world < 1 or R < 0:
        raise ValueError("bad ray sharding")
    q, r = divmod(R, world)
    out, lo = [], 0
    for k in range(world):
        hi = lo + q + (1 if k < r else 0)
        out.append((lo, hi))
        lo = hi
    return out


def ray_shards_weighted(work, world: int, ray_cost: float = 2.0):
    """Contiguous ray ranges [lo, hi) of the caller's ray order, one per rank, cut so
    that each holds about the same trace work: Σ (work[q] + ray_cost) over its rays,
    with work[q] the ray's band cells (Problem.ray_work) and ray_cost the per-ray
    setup and epilogue in cell equivalents.  Equal ray counts would leave the ranks
    holding edge detectors (rays leave the box sooner) with less work."""
    w = np.asarray(work, np.float64) + ray_cost
    R = len(w)
    if world < 1 or R < world:
        raise ValueError("bad ray sharding")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for k in range(1, world):
        c = int(np.searchsorted(cum, cum[-1] * k / world))
        cuts.append(min(max(c, cuts[-1] + 1), R - (world - k)))
    cuts.append(R)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def balanced_ray_shards(prob: dict, x0, world: int, device: int, measured: bool = True):
    """Ray shards of equal trace cost for state x0 ([P] host), from a temporary
    one-chain problem over all rays on `device`: measured=True cuts by the measured
    per-ray cost of the ray-lanes trace (Problem.ray_cost: SM cycles of each 32-ray
    warp task, divergence included; the band-cell count alone mispredicts it, see
    tools/shard_balance.py), else by band cells (Problem.ray_work)."""
    import torch
    from ._lib import Problem
    full = Problem(prob, device=device, max_chains=1)
    x = torch.from_numpy(np.ascontiguousarray(np.asarray(x0, np.float32).reshape(1, -1))).to(f"cuda:{device}")
    if measured:
        cost = full.ray_cost(x)
        for _ in range(2):   # the median of three measurements per ray
            cost = np.stack([cost, full.ray_cost(x)]) if cost.ndim == 1 else np.concatenate([cost, full.ray_cost(x)[None]])
        work = np.median(cost, axis=0)
        del full
        return ray_shards_weighted(work / max(float(np.mean(work)), 1e-30), world, ray_cost=0.0)
    work = full.ray_work(x)
    del full
    return ray_shards_weighted(work, world)


def ray_sharded_problem(prob: dict, rank: int, world: int, device: int, max_chains: int, group=None,
                        shards=None):
    """This rank's Problem over its ray shard with the in-library NCCL
    communicator attached (rank 0 creates the NCCL id; broadcast over the
    torch.distributed group).  shards: the ranges (e.g. balanced_ray_shards);
    default equal ray counts."""
    from ._lib import Problem, comm_unique_id
    lo, hi = (shards or ray_shards(len(prob["ray_det"]), world))[rank]
    pb = Problem(prob, device=device, max_chains=max_chains, ray_lo=lo, ray_hi=hi)
    if world > 1:
        import torch.distributed as dist
        obj = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        pb.attach_comm(obj[0], rank, world)
    return pb


def nested_rhat_from_partials(part: np.ndarray, n_super: int) -> np.ndarray:
    """Nested R̂ = sqrt(1 + B/W) per parameter from Σ m_k, Σ m_k², Σ W_k over all
    super-chains (mt_nested_rhat_partials summed over ranks)."""
    s1, s2, sw = part
    mean = s1 / n_super
    B = (s2 - n_super * mean ** 2) / (n_super - 1)
    W = sw / n_super
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.sqrt(1.0 + B / W)
    return np.where((W == 0) & (B <= 0), 1.0, r)


class ChainShard:
    """Device state of this rank's chains and the HMC loop.

    replicated=True: every rank holds the same chains (ray sharding) — the
    library all-reduces each evaluation, so acceptance and Welford statistics
    are already global and are not reduced again."""

    def __init__(self, problem, x0: np.ndarray, seed: int, L: int, eps0: float,
                 chain_offset: int = 0, n_chains_total: Optional[int] = None, group=None,
                 stream=None, replicated: bool = False, sampler: str = "hmc", max_depth: int = 8,
                 adapt_mass: bool = False):
        import torch
        self.torch = torch
        self.pb = problem
        self.dev = torch.device(f"cuda:{problem.device}")
        self.C, self.P = x0.shape
        self.seed, self.L = seed, L
        self.chain_offset = chain_offset
        self.n_total = n_chains_total or self.C
        self.group = group
        self.stream = stream
        # every torch-side operation on the shard's tensors runs on the shard's stream, in order
        # with the library calls it launches there (none when stream is None: the current stream)
        self._ctx = (lambda: torch.cuda.stream(stream)) if stream is not None else contextlib.nullcontext
        self.replicated = replicated
        if sampler not in ("hmc", "nuts"):
            raise ValueError(f"sampler {sampler!r}")
        self.sampler, self.max_depth = sampler, max_depth   # NUTS: 2^max_depth leaves cap
        self.adapt_mass = adapt_mass                        # diagonal mass from warm-up windows (R19b)
        self.minv = None
        with self._ctx():
            self._alloc(x0, eps0)
        self.n_samples = 0
        self.da = DualAveraging(eps0)
        self.it = 0
        problem.logpost_grad(self.x, self.logp, self.grad, self.status, stream=stream)

    def _alloc(self, x0, eps0):
        torch = self.torch
        t = lambda *s, dt=torch.float32: torch.zeros(s, dtype=dt, device=self.dev)  # noqa: E731
        self.x = torch.from_numpy(np.ascontiguousarray(x0, np.float32)).to(self.dev)
        self.logp = t(self.C, dt=torch.float64)
        self.grad = t(self.C, self.P)
        self.eps = torch.full((self.C,), eps0, dtype=torch.float32, device=self.dev)
        self.acc_prob = t(self.C)
        self.accepted = t(self.C, dt=torch.int32)
        self.depth = t(self.C, dt=torch.int32)
        self.status = t(self.C, dt=torch.int32)
        self.acc_fixed = t(2, dt=torch.int64)
        self.acc_mon = t(2, dt=torch.int64)      # sampling-phase acceptance sums (device, no host sync)
        self.mean = t(self.C, self.P)
        self.m2 = t(self.C, self.P)

    def refresh(self):
        """Re-evaluate logp / grad at the current x (after the problem's model changed)."""
        self.pb.logpost_grad(self.x, self.logp, self.grad, self.status, stream=self.stream)

    def _allreduce(self, t, op="sum"):
        if self.replicated:
            return t
        if self.group is not None or self._dist():
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=self.group)
        return t

    @staticmethod
    def _dist() -> bool:
        try:
            import torch.distributed as dist
            return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        except Exception:
            return False

    def step(self, adapt: bool = True, sample: bool = False, monitor: bool = False) -> float:
        """One HMC (or NUTS) iteration (a1-a9).  adapt: dual-averaging update of the global ε
        from the all-rank mean acceptance (one host read per iteration); returns that mean.
        monitor: add the acceptance sums to the device accumulator read by accept_rate() —
        no host synchronisation, so sampling iterations queue back to back.  sample: Welford."""
        pb = self.pb
        alpha = float("nan")
        with self._ctx():
            if self.sampler == "nuts":   # acc_prob <- the NUTS acceptance statistic
                pb.nuts_step(self.x, self.logp, self.grad, self.eps, self.max_depth, self.seed, self.it,
                             self.chain_offset, self.acc_prob, self.depth, self.accepted, self.status,
                             stream=self.stream)
            else:
                pb.hmc_step(self.x, self.logp, self.grad, self.eps, self.L, self.seed, self.it,
                            self.chain_offset, self.acc_prob, self.accepted, self.status, stream=self.stream)
            if adapt:
                self.acc_fixed.zero_()
                pb.stats_update(self.C, accept_prob=self.acc_prob, acc_fixed=self.acc_fixed, stream=self.stream)
            elif monitor:
                pb.stats_update(self.C, accept_prob=self.acc_prob, acc_fixed=self.acc_mon, stream=self.stream)
            if sample:
                pb.stats_update(self.C, x=self.x, n_prev=self.n_samples, mean=self.mean, m2=self.m2,
                                stream=self.stream)
                self.n_samples += 1
            if adapt:
                self._allreduce(self.acc_fixed)
                s, n = (int(v) for v in self.acc_fixed.cpu().tolist())
                alpha = s / 4294967296.0 / max(n, 1)
                self.eps.fill_(self.da.update(alpha))
        self.it += 1
        return alpha

    def step_graph(self, sample: bool = True, monitor: bool = True) -> None:
        """One sampling iteration (no adaptation), replayed from a CUDA graph: the
        step's ~4L + 5 launches reach the GPU as one graph launch, which matters where
        launches dominate (the small configs).  The Philox iteration and the Welford
        count live on the device (mt_set_step_counters) and advance inside the graph,
        so every replay is the next iteration and the results equal those of
        step(adapt=False, sample, monitor) bit for bit (tests/test_gpu_graph.py).
        HMC without a ray-shard communicator; the graph is captured on first use and
        again when the flags change.  launches_per_graph_step: the library launches
        one replay performs."""
        torch = self.torch
        if self.sampler != "hmc":
            raise ValueError("step_graph: HMC only")
        key = (sample, monitor)
        if getattr(self, "_graph_key", None) != key:
            if getattr(self, "_it_dev", None) is None:
                self._it_dev = torch.zeros(1, dtype=torch.int64, device=self.dev)
                self._n_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
            cur = torch.cuda.current_stream(self.dev) if self.stream is None else self.stream
            s = torch.cuda.Stream(device=self.dev)
            with torch.cuda.stream(cur):
                self._it_dev.fill_(self.it)
                self._n_dev.fill_(self.n_samples)
            s.wait_stream(cur)
            self.pb.set_step_counters(self._it_dev, self._n_dev)
            self.pb.timing_start(0)   # (counts the launches captured below; records no events)
            g = torch.cuda.CUDAGraph()
            # thread-local capture: other threads' CUDA calls (e.g. an NCCL process group's
            # watchdog under torchrun) must not invalidate the capture
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                self.pb.hmc_step(self.x, self.logp, self.grad, self.eps, self.L, self.seed, self.it,
                                 self.chain_offset, self.acc_prob, self.accepted, self.status, stream=s)
                if monitor:
                    self.pb.stats_update(self.C, accept_prob=self.acc_prob, acc_fixed=self.acc_mon, stream=s)
                if sample:
                    self.pb.stats_update(self.C, x=self.x, n_prev=self.n_samples, mean=self.mean, m2=self.m2,
                                         stream=s)
            self.launches_per_graph_step = self.pb.timing_read()["all_launches"]
            cur.wait_stream(s)
            self._graph, self._graph_key = g, key
        with self._ctx():
            self._graph.replay()
        self.it += 1
        if sample:
            self.n_samples += 1

    def accept_rate(self, reset: bool = True) -> float:
        """All-rank mean acceptance over the monitored iterations since the last reset
        (one host read)."""
        with self._ctx():
            tot = self._allreduce(self.acc_mon.clone())
            s, n = (int(v) for v in tot.cpu().tolist())
            if reset:
                self.acc_mon.zero_()
        return s / 4294967296.0 / max(n, 1)

    def end_warmup(self):
        with self._ctx():
            self.eps.fill_(self.da.final())

    def summary_update(self, nz: int = 60, gap: float = 10.0):
        """Accumulate the f4 posterior summaries of the current draws (mt_summary_update)."""
        if getattr(self, "_sum", None) is None:
            self._sum = (nz, gap) + tuple(self.pb.summary_buffers(nz))
        nz, gap, acc, mx, ml = self._sum
        self.pb.summary_update(self.x, self.logp, acc, nz, gap, mx, ml, stream=self.stream)

    def summaries(self):
        """Mean heights, air-gap probability, indicator-std tomography (all ranks'
        draws, all-reduced) and this rank's MAP draw."""
        nz, gap, acc, mx, ml = self._sum
        with self._ctx():
            acc = self._allreduce(acc.clone())
            out = self.pb.summaries(acc, nz)
            out.update(map_x=mx.cpu().numpy(), map_logp=float(ml.cpu()[0]), gap_threshold=gap)
        return out

    def nested_rhat(self, M: int = 8) -> np.ndarray:
        """Nested R̂ over super-chains of M contiguous chains."""
        with self._ctx():
            part = self.pb.nested_rhat_partials(self.C, M, self.mean, self.m2, max(self.n_samples, 1),
                                                stream=self.stream)
            self._allreduce(part)
            part = part.cpu().numpy()
        return nested_rhat_from_partials(part, self.n_total // M)

    def rhat(self) -> np.ndarray:
        with self._ctx():
            part = self.pb.rhat_partials(self.C, self.mean, self.m2, self.n_samples, stream=self.stream)
            self._allreduce(part)
            part = part.cpu().numpy()
        return rhat_from_partials(part, self.n_total, self.n_samples)

    def _mass_from_window(self, wmean, wm2, n: int):
        """Pooled within-chain variance of the window's draws -> regularised M^-1."""
        torch = self.torch
        with self._ctx():
            tot = torch.stack([wm2.sum(0).double(), torch.full((self.P,), float(self.C * (n - 1)),
                                                               dtype=torch.float64, device=self.dev)])
            self._allreduce(tot)
            var = tot[0] / tot[1]
            minv = (n / (n + 5.0)) * var + 1e-3 * (5.0 / (n + 5.0))
            self.minv = minv.float().contiguous()
            self.torch.cuda.current_stream().synchronize()   # (mt_set_inverse_mass copies synchronously)
            self.pb.set_inverse_mass(self.minv)

    def run(self, n_warmup: int, n_sample: int):
        accs = []
        windows = mass_windows(n_warmup) if self.adapt_mass else []
        wmean = wm2 = None
        for i in range(n_warmup):
            accs.append(self.step(adapt=True))
            for (a, b) in windows:
                if a <= i < b:
                    if i == a:
                        with self._ctx():
                            wmean = self.torch.zeros_like(self.x)
                            wm2 = self.torch.zeros_like(self.x)
                    self.pb.stats_update(self.C, x=self.x, n_prev=i - a, mean=wmean, m2=wm2, stream=self.stream)
                    if i == b - 1:   # window end: new mass, restart step-size adaptation (R19b)
                        self._mass_from_window(wmean, wm2, b - a)
                        self.da = DualAveraging(float(self.eps[0]))
        self.end_warmup()
        for _ in range(n_sample):
            self.step(adapt=False, sample=True)
        return dict(warmup_accept=accs, eps=float(self.eps[0]), rhat=self.rhat() if n_sample > 1 else None)
