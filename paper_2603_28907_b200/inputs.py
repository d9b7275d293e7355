"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NONE of the method's arithmetic (no ray tracing, no
opacity, no likelihood, no prior, no height map).  It only builds the
*instrument and scene description* the method consumes:

* the control-grid node coordinates ("grid of size
  n_rows x n_cols"; reading DESIGN.md R3: nodes at cell corners spanning the
  footprint, quantised to 2^-12 m),
* a synthetic "true" block-cave geometry given directly as node heights
  (stand-in for the expert model of P:162-185, which is not available;
  recipe in SURVEY.md §8(d.1) / DESIGN.md "Input recipe"),
* detectors and one ray per pixel centre (reading R10/R11),
* per-pixel solid-angle x efficiency weights ΔΩ_p·cos²θ_p (reading R9/R10:
  ε = cos²θ stand-in for the tables of Schouten 2022),
* seeded Gaussian perturbations for chain initial states.

Quantities that need the method itself (the flux calibration A, the observed
counts C_p = Poisson(λ_p(H_true)), and the latent x_true) are computed ONLY by
``tools/make_data.py`` through ``oracle/`` and stored in ``data/<config>.npz``.
"""
from __future__ import annotations

import dataclasses
import math
import os
from typing import Optional

import numpy as np

Q12 = 4096.0  # coordinates are multiples of 2^-12 m (R3/HP3)
DATA_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data")


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (configs[0..4])."""
    name: str
    n: int                      # control nodes per axis
    width: float                # footprint [0, width]^2 (m)
    det_layout: str             # "fixed" | "uniform_central" | "lattice"
    det_count: int              # detectors (lattice: per axis)
    n_theta: int
    n_phi: int
    theta_max_deg: float
    chains: int                 # chains per evaluation (chain_sharded: total over all GPUs)
    seed: int
    dome: bool
    z_top: float = 300.0        # reading R6: flat known Earth surface
    rho_muck: float = 1.90      # BASELINE.json configs[0] (g/cm^3)
    rho_air: float = 0.0012
    rho_rock: float = 2.65
    rho_ext: float = 2.65       # reading R7: rock beyond the footprint
    att_len: float = 250.0      # reading R9: Λ in g·cm^-3·m
    car_r: tuple = (0.95, 0.95)  # reading R13: fixed CAR r_ℓ (P:559-568 samples it; NEXT f2)
    median_lambda: float = 1000.0  # reading R9: exposure calibration target
    leapfrog_steps: int = 10    # configs[3]: 10 fused leapfrog steps
    hmc_iters: int = 200        # configs[3]: 200 iterations (100 warm-up)
    eps: float = 2e-3           # fixed-ε for trajectory parity (reading R20)

    @property
    def n_rays(self) -> int:
        return self.n_det * self.n_theta * self.n_phi

    @property
    def n_det(self) -> int:
        return self.det_count * self.det_count if self.det_layout == "lattice" else self.det_count

    @property
    def n_params(self) -> int:
        return 2 * self.n * self.n


CONFIGS = {
    "tiny": Config("tiny", 8, 100.0, "fixed", 1, 16, 16, 60.0, 4, 1, False),
    "small": Config("small", 16, 200.0, "uniform_central", 4, 64, 64, 60.0, 64, 2, False),
    "medium": Config("medium", 32, 400.0, "lattice", 4, 128, 128, 70.0, 1024, 3, True),
    "chain_sharded": Config("chain_sharded", 32, 400.0, "lattice", 4, 128, 128, 70.0, 8192, 3, True),
    "ray_sharded": Config("ray_sharded", 64, 800.0, "lattice", 8, 256, 256, 70.0, 1, 5, True),
}
# configs that share geometry/rays/data files
DATA_NAME = {"tiny": "tiny", "small": "small", "medium": "medium",
             "chain_sharded": "medium", "ray_sharded": "ray_sharded"}


def _streams(seed: int):
    """SeedSequence(seed).spawn(6) -> [truth, detectors, jitter, counts, chains, philox]."""
    ss = np.random.SeedSequence(seed).spawn(6)
    return [np.random.default_rng(s) for s in ss], ss


def quantize(v):
    return np.round(np.asarray(v, dtype=np.float64) * Q12) / Q12


def node_coords(cfg: Config) -> np.ndarray:
    """X_i = round(i·W/(n-1)·4096)/4096 (reading R3), exact in fp32."""
    i = np.arange(cfg.n, dtype=np.float64)
    return quantize(i * cfg.width / (cfg.n - 1)).astype(np.float32)


def truth_heights(cfg: Config) -> np.ndarray:
    """Synthetic true node heights [2][n][n] fp64 (ℓ=0 muck top, ℓ=1 cave back).

    Scene recipe (BASELINE.json configs[0]/[2]): cave back =
    150 m + 6-sinusoid field normalised to a 15 m peak; muck top = cave back −
    (5 m + softplus(N(0, 3²))); dome (+40 m cos² bump, radius 60 m) added to the
    cave back after the muck top is derived.  Scene synthesis only.
    """
    rngs, _ = _streams(cfg.seed)
    rt = rngs[0]
    X = node_coords(cfg).astype(np.float64)
    xx, yy = np.meshgrid(X, X, indexing="ij")  # [ix][iy]
    lam = rt.uniform(30.0, 80.0, size=6)
    alpha = rt.uniform(0.0, 2 * math.pi, size=6)
    phase = rt.uniform(0.0, 2 * math.pi, size=6)
    F = np.zeros_like(xx)
    for k in range(6):
        F += np.sin(2 * math.pi * (xx * math.cos(alpha[k]) + yy * math.sin(alpha[k])) / lam[k] + phase[k])
    f = 15.0 * F / np.max(np.abs(F))
    h1 = 150.0 + f
    xi = rt.normal(0.0, 3.0, size=xx.shape)
    h0 = h1 - (5.0 + np.logaddexp(0.0, xi))
    if cfg.dome:
        c = rt.uniform(cfg.width / 4, 3 * cfg.width / 4, size=2)
        rho = np.hypot(xx - c[0], yy - c[1])
        h1 = h1 + np.where(rho < 60.0, 40.0 * np.cos(math.pi * rho / (2 * 60.0)) ** 2, 0.0)
    H = np.stack([h0, h1])
    assert np.all(H[0] > 0) and np.all(H[1] > H[0]) and np.all(H[1] < cfg.z_top)
    return H


def detectors(cfg: Config) -> np.ndarray:
    """Detector positions [D][3] fp32 on the floor z=0, quantised to 2^-12 m."""
    rngs, _ = _streams(cfg.seed)
    W = cfg.width
    if cfg.det_layout == "fixed":
        xy = np.array([[W / 2, W / 2]])
    elif cfg.det_layout == "uniform_central":
        xy = rngs[1].uniform(W / 4, 3 * W / 4, size=(cfg.det_count, 2))
    elif cfg.det_layout == "lattice":
        k = cfg.det_count
        c = (np.arange(k) + 0.5) * (W / k)
        xx, yy = np.meshgrid(c, c, indexing="ij")
        xy = np.stack([xx.ravel(), yy.ravel()], axis=1)
        xy = xy + rngs[2].uniform(-W / (4 * k), W / (4 * k), size=xy.shape)
    else:
        raise ValueError(cfg.det_layout)
    xy = quantize(xy)
    return np.concatenate([xy, np.zeros((len(xy), 1))], axis=1).astype(np.float32)


def ray_grid(cfg: Config):
    """Pixel-centre rays, ordered detector -> θ -> φ (reading R11).

    Returns (ray_det int32 [R], ray_dir fp32 [R][3], w_unit fp64 [R]) where
    w_unit = ΔΩ_p·cos²θ_p (pixel solid angle × efficiency stand-in, R9/R10).
    """
    th_max = math.radians(cfg.theta_max_deg)
    nt, nph = cfg.n_theta, cfg.n_phi
    it = np.arange(nt, dtype=np.float64)
    th = (it + 0.5) * th_max / nt
    th_lo, th_hi = it * th_max / nt, (it + 1) * th_max / nt
    ph = (np.arange(nph, dtype=np.float64) + 0.5) * 2 * math.pi / nph
    dphi = 2 * math.pi / nph
    T, P = np.meshgrid(th, ph, indexing="ij")
    d = np.stack([np.sin(T) * np.cos(P), np.sin(T) * np.sin(P), np.cos(T)], axis=-1).reshape(-1, 3)
    dOmega = (dphi * (np.cos(th_lo) - np.cos(th_hi)))[:, None] * np.ones((1, nph))
    w_unit = (dOmega * np.cos(T) ** 2).reshape(-1)
    D = cfg.n_det
    ray_det = np.repeat(np.arange(D, dtype=np.int32), nt * nph)
    ray_dir = np.tile(d, (D, 1)).astype(np.float32)
    return ray_det, ray_dir, np.tile(w_unit, D)


def load_data(cfg: Config) -> Optional[dict]:
    path = os.path.join(DATA_DIR, DATA_NAME[cfg.name] + ".npz")
    if not os.path.exists(path):
        return None
    z = np.load(path)
    return {k: z[k] for k in z.files}


def make_problem(cfg_or_name, data: Optional[dict] = None) -> dict:
    """Canonical fp32 problem arrays (the single input contract of both sides).

    ``data`` (A, counts, x_true) defaults to ``data/<config>.npz`` written by
    tools/make_data.py via the oracle.  Without it the problem has A = 1 and
    zero counts (used only by make_data itself).
    """
    cfg = CONFIGS[cfg_or_name] if isinstance(cfg_or_name, str) else cfg_or_name
    if data is None:
        data = load_data(cfg)
    X = node_coords(cfg)
    ray_det, ray_dir, w_unit = ray_grid(cfg)
    A = float(data["A"]) if data is not None else 1.0
    counts = (data["counts"].astype(np.int32) if data is not None
              else np.zeros(len(ray_det), np.int32))
    prob = dict(
        name=cfg.name, cfg=cfg,
        node_x=X, node_y=X.copy(), z_top=np.float32(cfg.z_top),
        rho_muck=cfg.rho_muck, rho_air=cfg.rho_air, rho_rock=cfg.rho_rock, rho_ext=cfg.rho_ext,
        att_len=cfg.att_len, car_r=np.array(cfg.car_r, np.float32),
        det_xyz=detectors(cfg), ray_det=ray_det, ray_dir=ray_dir,
        ray_w=(A * w_unit).astype(np.float32), counts=counts, A=A,
        H_true=truth_heights(cfg),
    )
    if data is not None and "x_true" in data:
        prob["x_true"] = data["x_true"].astype(np.float64)
    return prob


def chain_states(x_true: np.ndarray, n_chains: int, seed: int, scale: float = 0.01,
                 chain_offset: int = 0, super_size: int = 1) -> np.ndarray:
    """Near-posterior initial states x = x_true + scale·ξ, fp32 [C][P].

    ξ ~ N(0, I) from the config's "chains" stream; chains of one super-chain
    (all components start from one state) share ξ.
    """
    rngs, _ = _streams(seed)
    P = x_true.size
    n_super = (chain_offset + n_chains + super_size - 1) // super_size
    xi = rngs[4].standard_normal((n_super, P))
    g = (np.arange(chain_offset, chain_offset + n_chains) // super_size)
    return (x_true.reshape(1, -1) + scale * xi[g]).astype(np.float32)


def prior_states(name: str, n_chains: int) -> np.ndarray:
    """fp32 [C][P] "prior-draw" chain states (wide active band, worst-case
    work), tiled from data/<config>_prior.npz (written by tools/make_data.py via the oracle)."""
    z = np.load(os.path.join(DATA_DIR, DATA_NAME[name] + "_prior.npz"))["x_prior"]
    return np.ascontiguousarray(z[np.arange(n_chains) % len(z)], dtype=np.float32)


def perturbed_heights(H: np.ndarray, n_chains: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """fp32 height fields [C][2][n][n] = H + scale·N(0,1) m, kept ordered.

    Used to feed BOTH sides the same heights (trace/adjoint parity without the
    latent map); H is a scene input, not a method output.
    """
    rng = np.random.default_rng(np.random.SeedSequence([seed, 77]))
    out = H[None] + scale * rng.standard_normal((n_chains,) + H.shape)
    out[:, 1] = np.maximum(out[:, 1], out[:, 0] + 0.5)
    return out.astype(np.float32)


def philox_key(cfg: Config) -> int:
    """64-bit Philox key for HMC: first 64 bits of the config's philox stream."""
    _, ss = _streams(cfg.seed)
    return int(ss[5].generate_state(1, dtype=np.uint64)[0])
