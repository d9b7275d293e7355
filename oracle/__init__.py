"""fp64 CPU oracle of the hot path (ctypes wrapper over oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke(), tools/make_data.py
and bench.py's cpu_baseline / ``--impl reference`` legs may import this
package.  The product path (paper_2603_28907_b200) never imports it.

Besides the C kernels this module holds the plain-Python parts of the oracle:
the leapfrog / HMC transition (readings R19/R20) and the inverse
heights map used by tools/make_data.py to place chains near the truth.
"""
from __future__ import annotations

import ctypes as ct
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (-O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", _SO, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ct.CDLL(_SO)
        L.or_problem_new.restype = ct.c_void_p
        L.or_problem_new.argtypes = [ct.c_int, ct.c_int, _fp, _fp, ct.c_float,
                                     ct.c_double, ct.c_double, ct.c_double, ct.c_double, ct.c_double,
                                     ct.c_double, ct.c_double, ct.c_int, _fp, ct.c_long,
                                     _ip, _fp, _fp, _ip]
        L.or_problem_free.argtypes = [ct.c_void_p]
        L.or_torus_spectrum.argtypes = [ct.c_int, ct.c_int, ct.c_double,
                                        ct.POINTER(ct.c_double), ct.POINTER(ct.c_double)]
        L.or_prior_surface.restype = ct.c_double
        L.or_prior_surface.argtypes = [ct.c_int, ct.c_int, ct.c_double, _dp, _dp]
        L.or_heights.argtypes = [ct.c_void_p, _dp, _dp, _dp]
        L.or_ray_extent.argtypes = [ct.c_void_p, ct.c_long, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double)]
        L.or_traversal.restype = ct.c_int
        L.or_traversal.argtypes = [ct.c_void_p, ct.c_long, _ip, _dp, _dp, ct.c_int]
        L.or_traversal_all.argtypes = [ct.c_void_p, ct.POINTER(ct.c_long), ct.c_void_p, ct.c_void_p]
        L.or_path_lengths.argtypes = [ct.c_void_p, ct.c_int, _dp, _dp, _dp, ct.c_void_p]
        L.or_loglik_grad_H.argtypes = [ct.c_void_p, ct.c_int, _dp, _dp, _dp, _dp, ct.c_void_p, _lp]
        L.or_logpost_grad.argtypes = [ct.c_void_p, ct.c_int, _dp, _dp, _dp, _dp, _dp, _dp,
                                      ct.c_void_p, _lp]
        L.or_torus_spectrum_dr.argtypes = [ct.c_int, ct.c_int, ct.c_double] + [ct.POINTER(ct.c_double)] * 4
        L.or_logpost_grad_r.argtypes = [ct.c_void_p, ct.c_int, _dp, _dp, _dp, _dp, _dp]
        L.or_ncp_kernel.argtypes = [ct.c_int, ct.c_int, ct.c_double, _dp, _dp]
        L.or_logpost_grad_ncp.argtypes = [ct.c_void_p, ct.c_int, _dp, _dp, _dp, _dp]
        L.or_voxel_path.restype = ct.c_int
        L.or_voxel_path.argtypes = [ct.c_void_p, ct.c_int, ct.c_long, _ip, _dp, ct.c_int]
        L.or_voxel_rhat.argtypes = [ct.c_void_p, ct.c_int, ct.c_double, _dp, ct.c_void_p, _dp]
        L.or_voxel_lambda.argtypes = [ct.c_void_p, ct.c_int, _dp, _dp]
        L.or_voxel_G_row.restype = ct.c_int
        L.or_voxel_G_row.argtypes = [ct.c_void_p, ct.c_int, _dp, ct.c_long, _ip, _dp, ct.c_int,
                                     ct.POINTER(ct.c_double)]
        L.or_voxel_logpost_grad.argtypes = [ct.c_void_p, ct.c_int, ct.c_double, ct.c_double, _dp,
                                            ct.c_int, _dp, _dp, _dp, _dp, _dp]
        L.or_philox4x32_10.argtypes = [_up, _up, _up]
        L.or_momenta.argtypes = [ct.c_int, ct.c_uint64, ct.c_uint64, ct.c_uint64, _dp]
        L.or_mh_uniform.restype = ct.c_double
        L.or_mh_uniform.argtypes = [ct.c_uint64, ct.c_uint64, ct.c_uint64]
        L.or_num_threads.restype = ct.c_int
        _lib = L
    return _lib


def num_threads() -> int:
    return lib().or_num_threads()


def torus_spectrum(nx: int, ny: int, r: float):
    """(σ, ln det Q) of the periodic CAR precision Q = diag(A1) - rA."""
    s, ld = ct.c_double(), ct.c_double()
    lib().or_torus_spectrum(nx, ny, r, ct.byref(s), ct.byref(ld))
    return s.value, ld.value


def torus_spectrum_dr(nx: int, ny: int, r: float):
    """(σ, dσ/dr, ln det Q, d ln det Q/dr) of the torus CAR precision Q(r) = 4I - rA."""
    out = [ct.c_double() for _ in range(4)]
    lib().or_torus_spectrum_dr(nx, ny, r, *[ct.byref(o) for o in out])
    return tuple(o.value for o in out)


def prior_surface(x: np.ndarray, r: float):
    """log N(x; 0, Q^-1) and its gradient for one [nx][ny] surface."""
    x = np.ascontiguousarray(x, np.float64)
    g = np.zeros_like(x)
    v = lib().or_prior_surface(x.shape[0], x.shape[1], r, x, g)
    return v, g


def prior_draws(nx: int, ny: int, r: float, n: int, rng) -> np.ndarray:
    """n draws of x ~ N(0, Q(r)^-1) on the n_x x n_y torus:
    Q = F* diag(λ) F with λ_ab = 4 - 2r(cos 2πa/n_x + cos 2πb/n_y), so
    x = Q^{-1/2} w = real(ifft2(fft2(w) / sqrt(λ))) for w ~ N(0, I).  -> [n][nx*ny]."""
    a = np.arange(nx)[:, None]
    b = np.arange(ny)[None, :]
    lam = 4.0 - 2.0 * r * (np.cos(2 * math.pi * a / nx) + np.cos(2 * math.pi * b / ny))
    w = rng.standard_normal((n, nx, ny))
    x = np.real(np.fft.ifft2(np.fft.fft2(w) / np.sqrt(lam)))
    return x.reshape(n, nx * ny)


def ncp_kernel(nx: int, ny: int, r: float):
    """(k, dk/dr) [nx][ny]: kernels of the circulant U = Q(r)^{-1/2} and dU/dr."""
    k = np.zeros(nx * ny)
    dk = np.zeros(nx * ny)
    lib().or_ncp_kernel(nx, ny, r, k, dk)
    return k.reshape(nx, ny), dk.reshape(nx, ny)


def philox4x32_10(ctr, key) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def momenta(P: int, seed: int, it: int, chain: int) -> np.ndarray:
    out = np.zeros(P, np.float64)
    lib().or_momenta(P, seed, it, chain, out)
    return out


def mh_uniform(seed: int, it: int, chain: int) -> float:
    return lib().or_mh_uniform(seed, it, chain)


class Problem:
    """The canonical fp32 problem (paper_2603_28907_b200.inputs.make_problem) in fp64."""

    def __init__(self, prob: dict):
        L = lib()
        self.prob = prob
        self.nx = len(prob["node_x"])
        self.ny = len(prob["node_y"])
        self.N = self.nx * self.ny
        self.P = 2 * self.N
        self.R = len(prob["ray_det"])
        self.z_top = float(prob["z_top"])
        self.car_r = [float(v) for v in prob["car_r"]]
        self._keep = [np.ascontiguousarray(prob[k]) for k in
                      ("node_x", "node_y", "det_xyz", "ray_det", "ray_dir", "ray_w", "counts")]
        nxa, nya, det, rdet, rdir, rw, cnt = self._keep
        self.h = L.or_problem_new(self.nx, self.ny, nxa.astype(np.float32), nya.astype(np.float32),
                                  float(prob["z_top"]), prob["rho_muck"], prob["rho_air"],
                                  prob["rho_rock"], prob["rho_ext"], prob["att_len"],
                                  self.car_r[0], self.car_r[1], len(det),
                                  np.ascontiguousarray(det, np.float32).ravel(), self.R,
                                  np.ascontiguousarray(rdet, np.int32),
                                  np.ascontiguousarray(rdir, np.float32).ravel(),
                                  np.ascontiguousarray(rw, np.float32),
                                  np.ascontiguousarray(cnt, np.int32))

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_problem_free(self.h)
            self.h = None

    # -- pieces ---------------------------------------------------------
    def sigma(self):
        return [torus_spectrum(self.nx, self.ny, r)[0] for r in self.car_r]

    def heights(self, x: np.ndarray):
        """x [2][nx][ny] -> (H [2][nx][ny], dH [3][nx][ny])."""
        x = np.ascontiguousarray(x, np.float64).reshape(2, self.nx, self.ny)
        H = np.zeros_like(x)
        dH = np.zeros((3, self.nx, self.ny))
        lib().or_heights(self.h, x, H, dH)
        return H, dH

    def ray_extent(self, q: int):
        s, le = ct.c_double(), ct.c_double()
        lib().or_ray_extent(self.h, q, ct.byref(s), ct.byref(le))
        return s.value, le.value

    def traversal(self, q: int):
        """[(i, j)] int32 [n][2], s_in [n], s_out [n]."""
        cap = 2 * (self.nx + self.ny) + 8
        ij = np.zeros(2 * cap, np.int32)
        si = np.zeros(cap)
        so = np.zeros(cap)
        n = lib().or_traversal(self.h, q, ij, si, so, cap)
        assert n <= cap
        return ij[:2 * n].reshape(n, 2), si[:n], so[:n]

    def traversal_all(self):
        """Every ray's traversal: off [R+1] (int64 CSR), ij [off[R]][2] int32, s_out [off[R]]."""
        off = np.zeros(self.R + 1, np.int64)
        lib().or_traversal_all(self.h, off.ctypes.data_as(ct.POINTER(ct.c_long)), None, None)
        ij = np.zeros((int(off[-1]), 2), np.int32)
        so = np.zeros(int(off[-1]))
        lib().or_traversal_all(self.h, off.ctypes.data_as(ct.POINTER(ct.c_long)), ij.ctypes.data, so.ctypes.data)
        return off, ij, so

    def path_lengths(self, H: np.ndarray, with_min_g1: bool = False):
        """H [C][2][nx][ny] -> L [C][R][3] (muck, air, rock), O [C][R] (, min|g'| [C][R])."""
        H = np.ascontiguousarray(H, np.float64).reshape(-1, 2, self.nx, self.ny)
        C = H.shape[0]
        L = np.zeros((C, self.R, 3))
        O = np.zeros((C, self.R))
        mg = np.zeros((C, self.R)) if with_min_g1 else None
        lib().or_path_lengths(self.h, C, H, L, O, mg.ctypes.data if with_min_g1 else None)
        return (L, O, mg) if with_min_g1 else (L, O)

    def loglik_grad_H(self, H: np.ndarray, with_sens: bool = False):
        """Per chain ll_dev, ll_std, dll/dH [C][2][nx][ny] (, sens) and work counters."""
        H = np.ascontiguousarray(H, np.float64).reshape(-1, 2, self.nx, self.ny)
        C = H.shape[0]
        ll = np.zeros(C)
        lls = np.zeros(C)
        G = np.zeros_like(H)
        sens = np.zeros(C)
        cnt = np.zeros(4, np.int64)
        lib().or_loglik_grad_H(self.h, C, H, ll, lls, G, sens.ctypes.data, cnt)
        out = dict(ll_dev=ll, ll_std=lls, dldH=G, counters=cnt)
        if with_sens:
            out["sens"] = sens
        return out

    def logpost_grad(self, x: np.ndarray):
        """x [C][P] -> dict(logp [C], grad [C][P], ll_dev, ll_std, prior, sens, counters)."""
        x = np.ascontiguousarray(x, np.float64).reshape(-1, self.P)
        C = x.shape[0]
        logp = np.zeros(C)
        g = np.zeros_like(x)
        ll = np.zeros(C)
        lls = np.zeros(C)
        pr = np.zeros(C)
        sens = np.zeros(C)
        cnt = np.zeros(4, np.int64)
        lib().or_logpost_grad(self.h, C, x, logp, g, ll, lls, pr, sens.ctypes.data, cnt)
        return dict(logp=logp, grad=g, ll_dev=ll, ll_std=lls, prior=pr, sens=sens, counters=cnt)

    def logpost_grad_r(self, v: np.ndarray):
        """Sampled r_l (f2): v [C][2N+2] = (x_0, x_1, ρ_0, ρ_1), r_l = logistic(ρ_l)
        -> dict(logp [C], grad [C][2N+2], ll_dev, prior)."""
        v = np.ascontiguousarray(v, np.float64).reshape(-1, self.P + 2)
        C = v.shape[0]
        logp, ll, pr = np.zeros(C), np.zeros(C), np.zeros(C)
        g = np.zeros_like(v)
        lib().or_logpost_grad_r(self.h, C, v, logp, g, ll, pr)
        return dict(logp=logp, grad=g, ll_dev=ll, prior=pr)

    # -- the paper's voxel / sigmoid / linearised model (f3, R28/R29)
    def voxel_path(self, nz: int, q: int):
        """Voxel ids and lengths of ray q's in-box segment."""
        cap = self.nx + self.ny + nz + 8
        vox = np.zeros(cap, np.int32)
        ln = np.zeros(cap)
        n = lib().or_voxel_path(self.h, nz, q, vox, ln, cap)
        assert n <= cap
        return vox[:n], ln[:n]

    def voxel_rhat(self, H: np.ndarray, nz: int, gamma: float = 1.0, with_weights: bool = False):
        """H [2][nx][ny] -> R̂ [n_grid] (, W [3][n_grid])."""
        H = np.ascontiguousarray(H, np.float64).reshape(-1)
        ng = self.N * nz
        Rh = np.zeros(ng)
        W = np.zeros(3 * ng) if with_weights else None
        lib().or_voxel_rhat(self.h, nz, gamma, H, W.ctypes.data if with_weights else None, Rh)
        return (Rh, W.reshape(3, ng)) if with_weights else Rh

    def voxel_lambda(self, R: np.ndarray, nz: int):
        """λ_p(R) for every ray, R [n_grid] piecewise constant."""
        lam = np.zeros(self.R)
        lib().or_voxel_lambda(self.h, nz, np.ascontiguousarray(R, np.float64), lam)
        return lam

    def voxel_G_row(self, R0: np.ndarray, nz: int, q: int):
        """(voxel ids, G_pv, λ_p(R0)) of row q of G = ∂λ/∂R at R0."""
        cap = self.nx + self.ny + nz + 8
        vox = np.zeros(cap, np.int32)
        g = np.zeros(cap)
        lam0 = ct.c_double()
        n = lib().or_voxel_G_row(self.h, nz, np.ascontiguousarray(R0, np.float64), q, vox, g, cap,
                                 ct.byref(lam0))
        return vox[:n], g[:n], lam0.value

    def voxel_logpost_grad(self, x: np.ndarray, Href: np.ndarray, nz: int, gamma: float = 1.0,
                           tau: float = 1e-3):
        """Linearised smooth model λ̂ = λ(R0) + G(R̂(H) - R0), R0 = R̂(H_ref) (P:293-294,
        P:386-390) -> dict(logp, grad, ll_dev, prior)."""
        x = np.ascontiguousarray(x, np.float64).reshape(-1, self.P)
        C = x.shape[0]
        logp, ll, pr = np.zeros(C), np.zeros(C), np.zeros(C)
        g = np.zeros_like(x)
        lib().or_voxel_logpost_grad(self.h, nz, gamma, tau,
                                    np.ascontiguousarray(Href, np.float64).reshape(-1), C, x, logp, g,
                                    ll, pr)
        return dict(logp=logp, grad=g, ll_dev=ll, prior=pr)

    def logpost_grad_ncp(self, v: np.ndarray):
        """Non-centred (f2): v [C][2N+2] = (z_0, z_1, ρ_0, ρ_1), x_l = U(r_l) z_l
        -> dict(logp [C], grad [C][2N+2], ll_dev)."""
        v = np.ascontiguousarray(v, np.float64).reshape(-1, self.P + 2)
        C = v.shape[0]
        logp, ll = np.zeros(C), np.zeros(C)
        g = np.zeros_like(v)
        lib().or_logpost_grad_ncp(self.h, C, v, logp, g, ll)
        return dict(logp=logp, grad=g, ll_dev=ll)

    def loglik_offset(self) -> float:
        """Σ_p (C ln C - C - ln Γ(C+1)): ll_std - ll_dev (R15)."""
        c = np.asarray(self.prob["counts"], np.float64)
        t = np.where(c > 0, c * np.log(np.where(c > 0, c, 1.0)), 0.0) - c
        from scipy.special import gammaln
        return float(np.sum(t - gammaln(c + 1.0)))

    # -- inverse map (for chain placement only) -------------------------
    def latent_from_heights(self, H: np.ndarray) -> np.ndarray:
        """x with heights(x) = H: x0 = σ0 Φ^-1(H0/z_top), x1 = σ1 Φ^-1((H1-H0)/(z_top-H0))."""
        from scipy.special import ndtri
        s = self.sigma()
        H = np.asarray(H, np.float64).reshape(2, self.nx, self.ny)
        x0 = s[0] * ndtri(H[0] / self.z_top)
        x1 = s[1] * ndtri((H[1] - H[0]) / (self.z_top - H[0]))
        return np.stack([x0, x1]).reshape(-1)


# ---------------------------------------------------------------------------
# Hamiltonian Monte Carlo.  Plain Python: velocity-Verlet with
# identity mass (R19), accept iff ln u < -ΔH (Metropolis correction).
# ---------------------------------------------------------------------------

def leapfrog(x, p, eps, L, logp_grad, minv=None):
    """L kick-drift-kick steps.  logp_grad(x [C][P]) -> (logp [C], grad [C][P]).

    eps: scalar or [C].  minv: diagonal inverse mass [P] (None: identity; R19b):
    drift x += ε M^-1 p.  Returns (x, p, logp, grad) after L steps.
    """
    x = np.array(x, np.float64)
    p = np.array(p, np.float64)
    mi = 1.0 if minv is None else np.asarray(minv, np.float64)
    e = np.asarray(eps, np.float64).reshape(-1, 1) if np.ndim(eps) else float(eps)
    lp, g = logp_grad(x)
    for _ in range(L):
        p = p + 0.5 * e * g
        x = x + e * mi * p
        lp, g = logp_grad(x)
        p = p + 0.5 * e * g
    return x, p, lp, g


def hmc_step(x, eps, L, logp_grad, seed, it, chain_offset=0, minv=None):
    """One HMC transition per chain with Philox momenta and MH uniforms; minv the
    diagonal inverse mass (p = z / sqrt(minv) ~ N(0, M), kinetic ½ pᵀ M^-1 p).

    Returns (x_new, accept_prob [C], accepted [C] bool, logp_new, dH [C]).
    """
    x = np.array(x, np.float64)
    C, P = x.shape
    mi = np.ones(P) if minv is None else np.asarray(minv, np.float64)
    p0 = np.stack([momenta(P, seed, it, chain_offset + c) for c in range(C)]) / np.sqrt(mi)
    lp0, _ = logp_grad(x)
    x1, p1, lp1, _ = leapfrog(x, p0, eps, L, logp_grad, minv)
    H0 = -lp0 + 0.5 * np.sum(mi * p0 * p0, axis=1)
    H1 = -lp1 + 0.5 * np.sum(mi * p1 * p1, axis=1)
    dH = H1 - H0
    u = np.array([mh_uniform(seed, it, chain_offset + c) for c in range(C)])
    with np.errstate(over="ignore", invalid="ignore"):
        acc_prob = np.where(np.isfinite(dH), np.minimum(1.0, np.exp(-dH)), 0.0)
    accepted = np.isfinite(dH) & (dH <= 1000.0) & (np.log(u) < -dH)
    x_new = np.where(accepted[:, None], x1, x)
    lp_new = np.where(accepted, lp1, lp0)
    return x_new, acc_prob, accepted, lp_new, dH


# ---------------------------------------------------------------------------
# No-U-Turn Sampler (NUTS of Hoffman & Gelman as run by NumPyro,
# trajectory capped at 2^max_depth leapfrog steps).  Plain Python,
# one chain at a time, in the order of the algorithm (reading R26 in DESIGN.md):
#   momenta p ~ N(0, I); the trajectory doubles max_depth times at most; at
#   depth j a direction v_j = ±1 is drawn and a subtree of 2^j leapfrog steps
#   is integrated from the tree's edge on that side with step v_j·ε;
#   within the subtree a leaf replaces the subtree proposal with probability
#   w_leaf / W_subtree (progressive multinomial sampling, w = e^{-ΔH});
#   the subtree is rejected (and the tree stops) on a divergence (ΔH > 1000
#   or non-finite) or a U-turn of any aligned sub-subtree (iterative checks
#   against checkpoints); a valid subtree's proposal replaces the tree's with
#   probability min(1, W_subtree / W_tree) (biased progressive sampling), then
#   the whole tree is checked for a U-turn between its two edge momenta;
#   U-turn(p⁻, p⁺, ρ): p⁻·(ρ - (p⁻+p⁺)/2) <= 0 or p⁺·(ρ - (p⁻+p⁺)/2) <= 0,
#   ρ = Σ momenta of the (sub)tree, identity mass.
# Random numbers: Philox4x32-10 word 0, counter (q, chain, iter, stream):
#   stream 2: direction at depth q (u >= 1/2 -> +1); stream 3: leaf q of the
#   iteration (within-subtree choice); stream 4: merge at depth q.
# ---------------------------------------------------------------------------

def philox_uniform(seed: int, it: int, chain: int, stream: int, q: int) -> float:
    w = philox4x32_10([q & 0xffffffff, chain & 0xffffffff, it & 0xffffffff, stream],
                      [seed & 0xffffffff, (seed >> 32) & 0xffffffff])
    return (float(w[0]) + 0.5) * 2.0 ** -32


def leaf_ckpt_idxs(n: int):
    """Checkpoint range for leaf n of a subtree: idx_max = popcount(n >> 1),
    idx_min = idx_max - (trailing ones of n) + 1."""
    idx_max = bin(n >> 1).count("1")
    t = 0
    while (n >> t) & 1:
        t += 1
    return idx_max - t + 1, idx_max


def is_turning(p_left, p_right, rho, minv=1.0):
    """Generalised U-turn on the velocities M^-1 p of the two ends."""
    rs = rho - 0.5 * (p_left + p_right)
    return float(np.dot(minv * p_left, rs)) <= 0.0 or float(np.dot(minv * p_right, rs)) <= 0.0


def nuts_step(x, lp, g, eps, logp_grad1, seed, it, chain, max_depth=8, trace=None, minv=None):
    """One NUTS transition of one chain.  logp_grad1(x [P]) -> (logp, grad [P]).
    Returns dict(x, logp, grad, depth, n_leaves, accept_stat, diverging).
    trace (a list, optional) receives (kind, margin, x) for every random choice:
    the distance of log u from its threshold (debugging threshold flips)."""
    x = np.array(x, np.float64)
    P = x.size
    mi = np.ones(P) if minv is None else np.asarray(minv, np.float64)
    p = momenta(P, seed, it, chain) / np.sqrt(mi)
    H0 = -lp + 0.5 * float(p @ (mi * p))
    left = right = (x, p, g, lp)                 # (θ, p, ∇, logp) of the two edges
    prop = (x, lp, g)
    logW = 0.0                                   # log Σ e^{-ΔH} over the tree (initial leaf: ΔH = 0)
    rho = p.copy()
    n_leaf, acc_sum, diverging, depth = 0, 0.0, False, 0
    for j in range(max_depth):
        v = 1 if philox_uniform(seed, it, chain, 2, j) >= 0.5 else -1
        th, pp, gg, ll = right if v > 0 else left
        logWs, rhos, props = -math.inf, np.zeros(P), None
        r_ck = [None] * (max_depth + 1)
        rs_ck = [None] * (max_depth + 1)
        ok = True
        for n in range(2 ** j):
            e = v * eps
            pp = pp + 0.5 * e * gg
            th = th + e * mi * pp
            ll, gg = logp_grad1(th)
            pp = pp + 0.5 * e * gg
            dH = (-ll + 0.5 * float(pp @ (mi * pp))) - H0
            acc_sum += min(1.0, math.exp(-dH)) if math.isfinite(dH) else 0.0
            n_leaf += 1
            if not math.isfinite(dH) or dH > 1000.0:
                ok, diverging = False, True
                break
            logWs_new = np.logaddexp(logWs, -dH)
            u = philox_uniform(seed, it, chain, 3, n_leaf - 1)
            if trace is not None:
                trace.append(("leaf", math.log(u) - (-dH - logWs_new), th))
            if math.log(u) < -dH - logWs_new:
                props = (th, ll, gg)
            logWs = logWs_new
            rhos = rhos + pp
            lo, hi = leaf_ckpt_idxs(n)
            if n % 2 == 0:
                r_ck[hi], rs_ck[hi] = pp, rhos.copy()
            else:
                for i in range(hi, lo - 1, -1):
                    if is_turning(r_ck[i], pp, rhos - rs_ck[i] + r_ck[i], mi):
                        ok = False
                        break
                if not ok:
                    break
        depth = j + 1
        if not ok:
            break
        if trace is not None:
            trace.append(("merge", math.log(philox_uniform(seed, it, chain, 4, j)) - (logWs - logW), props[0]))
        if math.log(philox_uniform(seed, it, chain, 4, j)) < logWs - logW:
            prop = props
        logW = np.logaddexp(logW, logWs)
        if v > 0:
            right = (th, pp, gg, ll)
        else:
            left = (th, pp, gg, ll)
        rho = rho + rhos
        if is_turning(left[1], right[1], rho, mi):
            break
    return dict(x=prop[0], logp=prop[1], grad=prop[2], depth=depth, n_leaves=n_leaf,
                accept_stat=acc_sum / max(n_leaf, 1), diverging=diverging)


# ---------------------------------------------------------------------------
# Posterior summaries (reading R27 in DESIGN.md): plain numpy over a
# list of draw sets, each [C][P] with its log-posteriors [C].
# ---------------------------------------------------------------------------
def sigmoid(u, gamma=1.0):
    """ς_γ(u) = 1/(1 + e^{-u/γ})."""
    return 1.0 / (1.0 + np.exp(-np.asarray(u, np.float64) / gamma))


def layer_indicators(H0, H1, z_top, nz):
    """D^(l)_{ijk} = ς(H_l - kΔz) - ς(H_{l-1} - kΔz) for l = muck (H_{-1} = 0),
    air, rock (H_2 = z_top), voxel columns at the nodes, Δz = z_top/nz -> [3][nx][ny][nz]."""
    z = np.arange(nz) * (z_top / nz)
    b = [np.zeros_like(H0), H0, H1, np.full_like(H0, z_top)]
    s = [sigmoid(h[..., None] - z) for h in b]
    return np.stack([s[1] - s[0], s[2] - s[1], s[3] - s[2]])


def posterior_summaries(op, draws, logps, nz, gap):
    """MAP draw, mean heights, air-thickness exceedance
    probability, std across draws of the layer indicators."""
    Hs, Ds, best = [], [], (-math.inf, None)
    for xs, lps in zip(draws, logps):
        for x, lp in zip(np.asarray(xs, np.float64), lps):
            H = op.heights(x[:op.P])[0]
            Hs.append(H)
            Ds.append(layer_indicators(H[0], H[1], op.z_top, nz))
            if lp > best[0]:
                best = (float(lp), x)
    Hs, Ds = np.array(Hs), np.array(Ds)
    return dict(mean_heights=Hs.mean(0), gap_probability=((Hs[:, 1] - Hs[:, 0]) > gap).mean(0),
                indicator_std=Ds.std(0), map_logp=best[0], map_x=best[1], draws=len(Hs))
