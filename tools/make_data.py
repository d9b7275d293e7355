"""Write data/<config>.npz: flux calibration A, observed counts, latent truth.

Calls ONLY oracle/ (plus the seeded scene generator): every stored value is a
function of the synthetic truth H_true through the fp64 oracle.

* A = median_target / median_p λ_p(H_true; A=1)        (reading R9)
* C_p ~ Poisson(A·λ_p(H_true; A=1)), "counts" stream     (reading R12)
* x_true = inverse heights map of H_true

Usage: python tools/make_data.py [config ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2603_28907_b200 import inputs  # noqa: E402


def make(name: str):
    cfg = inputs.CONFIGS[name]
    prob = inputs.make_problem(cfg, data=None)       # A = 1, counts = 0
    op = oracle.Problem(prob)
    H = prob["H_true"]
    _, O = op.path_lengths(H[None])
    w1 = prob["ray_w"].astype(np.float64)             # fp32(A=1 weights)
    lam1 = w1 * np.exp(-O[0] / cfg.att_len)
    A = cfg.median_lambda / float(np.median(lam1))
    rngs, _ = inputs._streams(cfg.seed)
    # λ at the calibrated exposure, from the fp32 weights the problem will carry
    _, _, w_unit = inputs.ray_grid(cfg)
    lam = (A * w_unit).astype(np.float32).astype(np.float64) * np.exp(-O[0] / cfg.att_len)
    counts = rngs[3].poisson(lam)
    assert counts.max() < 65536
    x_true = op.latent_from_heights(H)
    out = os.path.join(inputs.DATA_DIR, name + ".npz")
    np.savez_compressed(out, A=np.float64(A), counts=counts.astype(np.uint16), x_true=x_true)
    print(f"{name}: R={op.R} A={A:.6g} counts[min,med,max]=[{counts.min()},{np.median(counts)},"
          f"{counts.max()}] x_true[{x_true.min():.3f},{x_true.max():.3f}] -> {out} "
          f"({os.path.getsize(out)} B)")


def make_prior_states(name: str, n: int = 128):
    """data/<config>_prior.npz: n chain states x = (x_0, x_1) drawn from the CAR prior
    N(0, Q(r_l)^-1) by oracle.prior_draws — the wide-band "prior-draw" set of SURVEY
    §8(d.1), used for worst-case work and parity far from the posterior."""
    cfg = inputs.CONFIGS[name]
    rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, 99]))
    x = np.concatenate([oracle.prior_draws(cfg.n, cfg.n, cfg.car_r[l], n, rng) for l in range(2)], axis=1)
    out = os.path.join(inputs.DATA_DIR, name + "_prior.npz")
    np.savez_compressed(out, x_prior=x.astype(np.float32))
    print(f"{name}: {n} prior-draw states x[{x.min():.3f},{x.max():.3f}] -> {out} ({os.path.getsize(out)} B)")


if __name__ == "__main__":
    names = sys.argv[1:] or ["tiny", "small", "medium", "ray_sharded"]
    for n in names:
        if n.endswith("_prior"):
            make_prior_states(n[:-len("_prior")])
        else:
            make(n)
