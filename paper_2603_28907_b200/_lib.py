"""Thin ctypes binding of libmt.so (include/mt.h).  Argument marshalling only:
every step of the hot path runs in the CUDA kernels behind the C ABI.  PyTorch
supplies device memory and streams.  There is no fallback: if libmt.so is
missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as ct
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("MT_LIB") or os.path.join(_HERE, "libmt.so")   # MT_LIB: tuning variants

MT_STATUS_NONFINITE = 1
MT_STATUS_DIVERGENT = 2


class MTError(RuntimeError):
    pass


class _Desc(ct.Structure):
    _fields_ = [
        ("n_x", ct.c_int32), ("n_y", ct.c_int32),
        ("node_x", ct.c_void_p), ("node_y", ct.c_void_p),
        ("z_top", ct.c_float),
        ("rho_muck", ct.c_float), ("rho_air", ct.c_float), ("rho_rock", ct.c_float), ("rho_ext", ct.c_float),
        ("att_len", ct.c_float),
        ("car_r", ct.c_float * 2),
        ("n_det", ct.c_int32), ("det_xyz", ct.c_void_p),
        ("n_rays", ct.c_int64), ("ray_det", ct.c_void_p), ("ray_dir", ct.c_void_p),
        ("ray_w", ct.c_void_p), ("counts", ct.c_void_p),
        ("ray_lo", ct.c_int64), ("ray_hi", ct.c_int64),
        ("device", ct.c_int32), ("max_chains", ct.c_int32), ("sample_r", ct.c_int32),
        ("noncentred", ct.c_int32),
    ]


EXPORTS = [
    "mt_problem_create", "mt_problem_destroy", "mt_num_params", "mt_num_rays", "mt_loglik_offset",
    "mt_prior_constants", "mt_logpost_grad", "mt_leapfrog", "mt_draw_momenta", "mt_hmc_step",
    "mt_stats_update", "mt_rhat_partials", "mt_heights", "mt_loglik_heights", "mt_path_lengths", "mt_debug_traversal", "mt_traversal_all", "mt_ray_work", "mt_ray_cost", "mt_nuts_record", "mt_philox",
    "mt_philox_curand", "mt_timing_start", "mt_timing_read", "mt_trace_counters", "mt_measure_fp32_peak",
    "mt_last_error", "mt_comm_unique_id", "mt_attach_comm", "mt_detach_comm", "mt_nuts_step",
    "mt_nested_rhat_partials", "mt_summary_update", "mt_summary_finalize", "mt_set_step_counters",
    "mt_voxel_model", "mt_voxel_info",
    "mt_voxel_counters", "mt_measure_l2_gather", "mt_set_inverse_mass",
]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise MTError(f"{SO_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ct.CDLL(SO_PATH)
        vp, i32, i64, u32, u64, dbl = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_uint32, ct.c_uint64, ct.c_double
        sig = {
            "mt_problem_create": ([ct.POINTER(_Desc), ct.POINTER(vp)], ct.c_int),
            "mt_problem_destroy": ([vp], ct.c_int),
            "mt_num_params": ([vp], i32),
            "mt_num_rays": ([vp], i64),
            "mt_loglik_offset": ([vp], dbl),
            "mt_prior_constants": ([vp, vp, vp], ct.c_int),
            "mt_logpost_grad": ([vp, i32, vp, vp, vp, vp, vp], ct.c_int),
            "mt_leapfrog": ([vp, i32, vp, vp, vp, vp, vp, i32, vp], ct.c_int),
            "mt_draw_momenta": ([vp, i32, vp, u64, u64, u64, vp], ct.c_int),
            "mt_hmc_step": ([vp, i32, vp, vp, vp, vp, i32, u64, u64, u64, vp, vp, vp, vp], ct.c_int),
            "mt_stats_update": ([vp, i32, vp, vp, i32, vp, vp, vp, vp], ct.c_int),
            "mt_rhat_partials": ([vp, i32, vp, vp, i32, vp, vp], ct.c_int),
            "mt_nested_rhat_partials": ([vp, i32, i32, vp, vp, i32, vp, vp], ct.c_int),
            "mt_summary_update": ([vp, i32, vp, vp, i32, ct.c_float, vp, vp, vp, vp], ct.c_int),
            "mt_summary_finalize": ([vp, i32, vp, vp, vp], ct.c_int),
            "mt_set_step_counters": ([vp, vp, vp], ct.c_int),
            "mt_heights": ([vp, i32, vp, vp, vp], ct.c_int),
            "mt_loglik_heights": ([vp, i32, vp, vp, vp, vp], ct.c_int),
            "mt_path_lengths": ([vp, i32, vp, vp, vp, vp], ct.c_int),
            "mt_debug_traversal": ([vp, i64, vp, vp, vp, i32, vp], ct.c_int),
            "mt_traversal_all": ([vp, vp, vp, vp], ct.c_int),
            "mt_ray_work": ([vp, vp, vp], ct.c_int),
            "mt_ray_cost": ([vp, vp, vp], ct.c_int),
            "mt_nuts_record": ([vp, vp, vp, vp, i32], ct.c_int),
            "mt_philox": ([vp, u32, u32, vp, i64, vp], ct.c_int),
            "mt_philox_curand": ([vp, u32, u32, vp, i64, vp], ct.c_int),
            "mt_timing_start": ([vp, i32], ct.c_int),
            "mt_timing_read": ([vp, vp, vp, vp, vp], ct.c_int),
            "mt_trace_counters": ([vp, vp, vp], ct.c_int),
            "mt_comm_unique_id": ([vp], ct.c_int),
            "mt_nuts_step": ([vp, i32, vp, vp, vp, vp, i32, u64, u64, u64, vp, vp, vp, vp, vp], ct.c_int),
            "mt_attach_comm": ([vp, vp, i32, i32], ct.c_int),
            "mt_detach_comm": ([vp], ct.c_int),
            "mt_measure_fp32_peak": ([i32, vp, vp], ct.c_int),
            "mt_voxel_model": ([vp, i32, ct.c_float, ct.c_float, vp], ct.c_int),
            "mt_voxel_info": ([vp, vp, vp, vp], ct.c_int),
            "mt_voxel_counters": ([vp, vp], ct.c_int),
            "mt_set_inverse_mass": ([vp, vp, i32], ct.c_int),
            "mt_measure_l2_gather": ([i32, i64, vp], ct.c_int),
            "mt_last_error": ([], ct.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().mt_last_error().decode(errors="replace")
        raise MTError(f"{what} failed (code {rc}): {msg}")


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _dev_tensor(t, dtype, shape, device, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise MTError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise MTError(f"{name} must be contiguous {dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise MTError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.device.index != device:
        raise MTError(f"{name} is on cuda:{t.device.index}, problem on cuda:{device}")
    return t


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ct.c_void_p(s.cuda_stream)


class Problem:
    """A canonical problem bound to one CUDA device (mt_problem_create)."""

    def __init__(self, prob: dict, device: int = 0, max_chains: int = 1,
                 ray_lo: int = 0, ray_hi: Optional[int] = None, sample_r: bool = False,
                 noncentred: bool = False):
        self._keep = {
            "node_x": np.ascontiguousarray(prob["node_x"], np.float32),
            "node_y": np.ascontiguousarray(prob["node_y"], np.float32),
            "det_xyz": np.ascontiguousarray(prob["det_xyz"], np.float32),
            "ray_det": np.ascontiguousarray(prob["ray_det"], np.int32),
            "ray_dir": np.ascontiguousarray(prob["ray_dir"], np.float32),
            "ray_w": np.ascontiguousarray(prob["ray_w"], np.float32),
            "counts": np.ascontiguousarray(prob["counts"], np.int32),
        }
        k = self._keep
        R = len(k["ray_det"])
        d = _Desc()
        d.n_x, d.n_y = len(k["node_x"]), len(k["node_y"])
        d.node_x, d.node_y = k["node_x"].ctypes.data, k["node_y"].ctypes.data
        d.z_top = float(prob["z_top"])
        d.rho_muck, d.rho_air = float(prob["rho_muck"]), float(prob["rho_air"])
        d.rho_rock, d.rho_ext = float(prob["rho_rock"]), float(prob["rho_ext"])
        d.att_len = float(prob["att_len"])
        d.car_r[0], d.car_r[1] = float(prob["car_r"][0]), float(prob["car_r"][1])
        d.n_det = len(k["det_xyz"])
        d.det_xyz = k["det_xyz"].ctypes.data
        d.n_rays = R
        d.ray_det, d.ray_dir = k["ray_det"].ctypes.data, k["ray_dir"].ctypes.data
        d.ray_w, d.counts = k["ray_w"].ctypes.data, k["counts"].ctypes.data
        d.ray_lo = ray_lo
        d.ray_hi = R if ray_hi is None else ray_hi
        d.device = device
        d.max_chains = max_chains
        d.sample_r = 1 if (sample_r or noncentred) else 0
        d.noncentred = 1 if noncentred else 0
        h = ct.c_void_p()
        _check(lib().mt_problem_create(ct.byref(d), ct.byref(h)), "mt_problem_create")
        self.h = h
        self.device = device
        self.max_chains = max_chains
        self.nx, self.ny = d.n_x, d.n_y
        self.P = lib().mt_num_params(h)
        self.R = lib().mt_num_rays(h)
        self.loglik_offset = lib().mt_loglik_offset(h)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().mt_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prior_constants(self):
        s = (ct.c_double * 2)()
        ld = (ct.c_double * 2)()
        _check(lib().mt_prior_constants(self.h, s, ld), "mt_prior_constants")
        return list(s), list(ld)

    # -- hot path ----------------------------------------------------------
    def logpost_grad(self, x, logp=None, grad=None, status=None, stream=None):
        import torch
        C = x.shape[0]
        _dev_tensor(x, torch.float32, (C, self.P), self.device, "x")
        if logp is None:
            logp = torch.empty(C, dtype=torch.float64, device=x.device)
        if grad is None:
            grad = torch.empty_like(x)
        _check(lib().mt_logpost_grad(self.h, C, _ptr(x), _ptr(logp), _ptr(grad), _ptr(status),
                                     _stream(stream)), "mt_logpost_grad")
        return logp, grad

    def leapfrog(self, x, p, logp, grad, eps, L: int, stream=None):
        import torch
        C = x.shape[0]
        for t, n, dt, sh in ((x, "x", torch.float32, (C, self.P)), (p, "p", torch.float32, (C, self.P)),
                             (logp, "logp", torch.float64, (C,)), (grad, "grad", torch.float32, (C, self.P)),
                             (eps, "eps", torch.float32, (C,))):
            _dev_tensor(t, dt, sh, self.device, n)
        _check(lib().mt_leapfrog(self.h, C, _ptr(x), _ptr(p), _ptr(logp), _ptr(grad), _ptr(eps), L,
                                 _stream(stream)), "mt_leapfrog")

    def draw_momenta(self, C: int, seed: int, it: int, chain_offset: int = 0, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((C, self.P), dtype=torch.float32, device=f"cuda:{self.device}")
        _check(lib().mt_draw_momenta(self.h, C, _ptr(out), seed, it, chain_offset, _stream(stream)),
               "mt_draw_momenta")
        return out

    def hmc_step(self, x, logp, grad, eps, L: int, seed: int, it: int, chain_offset: int = 0,
                 accept_prob=None, accepted=None, status=None, stream=None):
        import torch
        C = x.shape[0]
        dev = x.device
        if accept_prob is None:
            accept_prob = torch.empty(C, dtype=torch.float32, device=dev)
        if accepted is None:
            accepted = torch.empty(C, dtype=torch.int32, device=dev)
        for t, n, dt, sh in ((x, "x", torch.float32, (C, self.P)), (logp, "logp", torch.float64, (C,)),
                             (grad, "grad", torch.float32, (C, self.P)), (eps, "eps", torch.float32, (C,))):
            _dev_tensor(t, dt, sh, self.device, n)
        _check(lib().mt_hmc_step(self.h, C, _ptr(x), _ptr(logp), _ptr(grad), _ptr(eps), L, seed, it,
                                 chain_offset, _ptr(accept_prob), _ptr(accepted), _ptr(status),
                                 _stream(stream)), "mt_hmc_step")
        return accept_prob, accepted

    def nuts_step(self, x, logp, grad, eps, max_depth: int, seed: int, it: int, chain_offset: int = 0,
                  accept_stat=None, depth=None, n_leaves=None, status=None, stream=None):
        """One NUTS transition per chain (mt_nuts_step); returns (accept_stat, depth, n_leaves)."""
        import torch
        C = x.shape[0]
        dev = x.device
        if accept_stat is None:
            accept_stat = torch.empty(C, dtype=torch.float32, device=dev)
        if depth is None:
            depth = torch.empty(C, dtype=torch.int32, device=dev)
        if n_leaves is None:
            n_leaves = torch.empty(C, dtype=torch.int32, device=dev)
        for t, n, dt, sh in ((x, "x", torch.float32, (C, self.P)), (logp, "logp", torch.float64, (C,)),
                             (grad, "grad", torch.float32, (C, self.P)), (eps, "eps", torch.float32, (C,))):
            _dev_tensor(t, dt, sh, self.device, n)
        _check(lib().mt_nuts_step(self.h, C, _ptr(x), _ptr(logp), _ptr(grad), _ptr(eps), max_depth, seed, it,
                                  chain_offset, _ptr(accept_stat), _ptr(depth), _ptr(n_leaves), _ptr(status),
                                  _stream(stream)), "mt_nuts_step")
        return accept_stat, depth, n_leaves

    def stats_update(self, C: int, x=None, accept_prob=None, n_prev: int = 0, mean=None, m2=None,
                     acc_fixed=None, stream=None):
        """a9: fixed-point acceptance sums (int64 [2]) and Welford mean/M2 of x."""
        _check(lib().mt_stats_update(self.h, C, _ptr(x), _ptr(accept_prob), n_prev, _ptr(mean), _ptr(m2),
                                     _ptr(acc_fixed), _stream(stream)), "mt_stats_update")

    def set_step_counters(self, iter_dev=None, n_prev_dev=None):
        """Device step counters for CUDA-graph capture (mt_set_step_counters): int64 [1]
        Philox iteration read and advanced by mt_hmc_step, int32 [1] Welford count read
        and advanced by mt_stats_update; None restores the host arguments."""
        import torch
        if iter_dev is not None:
            _dev_tensor(iter_dev, torch.int64, (1,), self.device, "iter")
        if n_prev_dev is not None:
            _dev_tensor(n_prev_dev, torch.int32, (1,), self.device, "n_prev")
        _check(lib().mt_set_step_counters(self.h, _ptr(iter_dev), _ptr(n_prev_dev)), "mt_set_step_counters")

    def rhat_partials(self, C: int, mean, m2, n: int, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((3, self.P), dtype=torch.float64, device=mean.device)
        _check(lib().mt_rhat_partials(self.h, C, _ptr(mean), _ptr(m2), n, _ptr(out), _stream(stream)),
               "mt_rhat_partials")
        return out

    def nested_rhat_partials(self, C: int, M: int, mean, m2, n: int, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((3, self.P), dtype=torch.float64, device=mean.device)
        _check(lib().mt_nested_rhat_partials(self.h, C, M, _ptr(mean), _ptr(m2), n, _ptr(out), _stream(stream)),
               "mt_nested_rhat_partials")
        return out

    def summary_update(self, x, logp, acc, nz: int, gap: float, map_x=None, map_logp=None, stream=None):
        """f4 posterior-summary accumulators (mt_summary_update); acc from summary_buffers()."""
        C = x.shape[0]
        _check(lib().mt_summary_update(self.h, C, _ptr(x), _ptr(logp), nz, gap, _ptr(acc), _ptr(map_x),
                                       _ptr(map_logp), _stream(stream)), "mt_summary_update")

    def summary_buffers(self, nz: int):
        import torch
        N = self.nx * self.ny
        dev = f"cuda:{self.device}"
        acc = torch.zeros(1 + 3 * N + 6 * N * nz, dtype=torch.float64, device=dev)
        return acc, torch.zeros(self.P, dtype=torch.float32, device=dev), \
            torch.full((1,), float("-inf"), dtype=torch.float64, device=dev)

    def summaries(self, acc, nz: int, stream=None):
        """Mean heights [2][nx][ny], air-gap exceedance probability [nx][ny] and
        indicator std [3][nx][ny][nz], assembled on the device by
        mt_summary_finalize."""
        import torch
        N = self.nx * self.ny
        out = torch.empty(3 * N * (1 + nz), dtype=torch.float64, device=acc.device)
        _check(lib().mt_summary_finalize(self.h, nz, _ptr(acc), _ptr(out), _stream(stream)), "mt_summary_finalize")
        o = out.cpu().numpy()
        return dict(mean_heights=o[:2 * N].reshape(2, self.nx, self.ny),
                    gap_probability=o[2 * N:3 * N].reshape(self.nx, self.ny),
                    indicator_std=o[3 * N:].reshape(3, self.nx, self.ny, nz), draws=int(acc[0].item()))

    # -- parity / debug ------------------------------------------------------
    def heights(self, x, stream=None):
        import torch
        C = x.shape[0]
        _dev_tensor(x, torch.float32, (C, self.P), self.device, "x")
        H = torch.empty((C, 2 * self.nx * self.ny), dtype=torch.float32, device=x.device)
        _check(lib().mt_heights(self.h, C, _ptr(x), _ptr(H), _stream(stream)), "mt_heights")
        return H.view(C, 2, self.nx, self.ny)

    def loglik_heights(self, H, stream=None):
        import torch
        C = H.shape[0]
        NH = 2 * self.nx * self.ny
        H = H.reshape(C, NH)
        _dev_tensor(H, torch.float32, (C, NH), self.device, "H")
        ll = torch.empty(C, dtype=torch.float64, device=H.device)
        G = torch.empty_like(H)
        _check(lib().mt_loglik_heights(self.h, C, _ptr(H), _ptr(ll), _ptr(G), _stream(stream)),
               "mt_loglik_heights")
        return ll, G.view(C, 2, self.nx, self.ny)

    def path_lengths(self, H, stream=None):
        import torch
        C = H.shape[0]
        NH = 2 * self.nx * self.ny
        H = H.reshape(C, NH)
        _dev_tensor(H, torch.float32, (C, NH), self.device, "H")
        L = torch.empty((C, self.R, 3), dtype=torch.float32, device=H.device)
        O = torch.empty((C, self.R), dtype=torch.float32, device=H.device)
        _check(lib().mt_path_lengths(self.h, C, _ptr(H), _ptr(L), _ptr(O), _stream(stream)),
               "mt_path_lengths")
        return L, O

    def ray_work(self, x) -> np.ndarray:
        """Per-ray trace work (band cells) for one chain state x (device [P]): int32 [R],
        caller's ray order (mt_ray_work; ray-shard balancing)."""
        out = np.zeros(self.R, np.int32)
        _check(lib().mt_ray_work(self.h, _ptr(x), out.ctypes.data), "mt_ray_work")
        return out

    def nuts_record(self, th=None, g=None, lp=None):
        """Record every leaf of the following nuts_step calls into th [K][C][P], g [K][C][P]
        (float32) and lp [K][C] (float64) device tensors (mt_nuts_record); no args: off."""
        if th is None:
            _check(lib().mt_nuts_record(self.h, None, None, None, 0), "mt_nuts_record")
            return
        _check(lib().mt_nuts_record(self.h, _ptr(th), _ptr(g), _ptr(lp), th.shape[0]), "mt_nuts_record")

    def ray_cost(self, x) -> np.ndarray:
        """Measured trace cost per ray (SM cycles, float32 [R], caller's ray order) for one
        chain state x (device [P]) on the ray-lanes trace (mt_ray_cost)."""
        out = np.zeros(self.R, np.float32)
        _check(lib().mt_ray_cost(self.h, _ptr(x), out.ctypes.data), "mt_ray_cost")
        return out

    def traversal_all(self):
        """Every ray's stored traversal in the caller's ray order: off [R+1] int64 (CSR),
        ij [off[R]][2] int32, s_out [off[R]] fp32 (mt_traversal_all; host, synchronous)."""
        off = np.zeros(self.R + 1, np.int64)
        _check(lib().mt_traversal_all(self.h, off.ctypes.data, None, None), "mt_traversal_all")
        ij = np.zeros((int(off[-1]), 2), np.int32)
        so = np.zeros(int(off[-1]), np.float32)
        _check(lib().mt_traversal_all(self.h, off.ctypes.data, ij.ctypes.data, so.ctypes.data), "mt_traversal_all")
        return off, ij, so

    def debug_traversal(self, ray: int, cap: Optional[int] = None):
        cap = cap or 2 * (self.nx + self.ny) + 8
        ij = np.zeros(2 * cap, np.int32)
        si = np.zeros(cap, np.float32)
        so = np.zeros(cap, np.float32)
        n = ct.c_int32()
        _check(lib().mt_debug_traversal(self.h, ray, ij.ctypes.data, si.ctypes.data, so.ctypes.data,
                                        cap, ct.byref(n)), "mt_debug_traversal")
        m = n.value
        assert m <= cap
        return ij[:2 * m].reshape(m, 2), si[:m], so[:m]

    # -- measurement ------------------------------------------------------------
    def timing_start(self, max_records: int = 4096):
        _check(lib().mt_timing_start(self.h, max_records), "mt_timing_start")

    def timing_read(self):
        ms, n, pairs, alln = ct.c_double(), ct.c_int64(), ct.c_double(), ct.c_int64()
        _check(lib().mt_timing_read(self.h, ct.byref(ms), ct.byref(n), ct.byref(pairs), ct.byref(alln)),
               "mt_timing_read")
        return dict(trace_ms=ms.value, trace_launches=n.value, pairs=pairs.value, all_launches=alln.value)

    def attach_comm(self, uid: bytes, rank: int, world: int):
        """Create the in-library NCCL communicator for ray sharding (collective over
        `world` ranks; uid from comm_unique_id() on one rank, broadcast by the caller)."""
        if len(uid) != 128:
            raise MTError("NCCL unique id must be 128 bytes")
        buf = ct.create_string_buffer(uid, 128)
        _check(lib().mt_attach_comm(self.h, buf, rank, world), "mt_attach_comm")

    def detach_comm(self):
        _check(lib().mt_detach_comm(self.h), "mt_detach_comm")

    def voxel_model(self, n_z: int, H_ref=None, gamma: float = 1.0, tau: float = 1e-3):
        """Switch to the paper's voxel / sigmoid / linearised model (mt_voxel_model,
        P:242-390) around R0 = R̂(H_ref), H_ref host [2][nx][ny]; n_z = 0 switches back."""
        import numpy as np
        if n_z == 0:
            _check(lib().mt_voxel_model(self.h, 0, 1.0, 0.0, None), "mt_voxel_model")
            return
        Hr = np.ascontiguousarray(np.asarray(H_ref, np.float32).reshape(2 * self.nx * self.ny))
        _check(lib().mt_voxel_model(self.h, n_z, gamma, tau, Hr.ctypes.data), "mt_voxel_model")

    def voxel_info(self):
        nz, nnz, ng = ct.c_int32(), ct.c_int64(), ct.c_int64()
        _check(lib().mt_voxel_info(self.h, ct.byref(nz), ct.byref(nnz), ct.byref(ng)), "mt_voxel_info")
        return dict(n_z=nz.value, nnz=nnz.value, n_grid=ng.value)

    def set_inverse_mass(self, minv=None):
        """Diagonal inverse mass M^-1 [P] (device fp32) for HMC / NUTS; None = identity."""
        import torch
        if minv is None:
            _check(lib().mt_set_inverse_mass(self.h, None, 0), "mt_set_inverse_mass")
            return
        _dev_tensor(minv, torch.float32, (self.P,), self.device, "minv")
        _check(lib().mt_set_inverse_mass(self.h, _ptr(minv), self.P), "mt_set_inverse_mass")

    def voxel_gathered_bytes(self) -> int:
        v = ct.c_uint64()
        _check(lib().mt_voxel_counters(self.h, ct.byref(v)), "mt_voxel_counters")
        return v.value

    def trace_counters(self):
        """Cumulative deferred chain x ray pairs (fp64 follow-up kernel) and the
        device time of the follow-up launches in the last timed region (ms)."""
        n, ms = ct.c_int64(), ct.c_double()
        _check(lib().mt_trace_counters(self.h, ct.byref(n), ct.byref(ms)), "mt_trace_counters")
        return dict(deferred=n.value, defer_ms=ms.value)


def comm_unique_id() -> bytes:
    """An NCCL unique id (128 bytes) for Problem.attach_comm."""
    buf = ct.create_string_buffer(128)
    _check(lib().mt_comm_unique_id(buf), "mt_comm_unique_id")
    return buf.raw


def philox(ctr, key, use_curand: bool = False, stream=None):
    """Raw Philox4x32-10 words for device counters ctr [n][4] (uint32 as int32 tensor)."""
    import torch
    n = ctr.shape[0]
    out = torch.empty_like(ctr)
    f = lib().mt_philox_curand if use_curand else lib().mt_philox
    _check(f(_ptr(ctr), key[0], key[1], _ptr(out), n, _stream(stream)), "mt_philox")
    return out


def measure_fp32_peak(device: int = 0):
    tf, mhz = ct.c_double(), ct.c_double()
    _check(lib().mt_measure_fp32_peak(device, ct.byref(tf), ct.byref(mhz)), "mt_measure_fp32_peak")
    return tf.value, mhz.value


def measure_l2_gather(device: int = 0, nbytes: int = 32 << 20) -> float:
    """Measured L2-resident 512-B-row gather bandwidth (GB/s), the voxel kernels' roofline."""
    v = ct.c_double()
    _check(lib().mt_measure_l2_gather(device, nbytes, ct.byref(v)), "mt_measure_l2_gather")
    return v.value
