"""Find the worst path-length pair of a config (CUDA vs oracle, identical
heights) and dump that ray: traversal (device vs oracle), band, per-unit
lengths.  Debugging aid; test infrastructure (imports oracle/).

  python tools/debug_ray.py <config> [chains]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2603_28907_b200 import Problem, inputs  # noqa: E402


def main():
    name = sys.argv[1]
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    prob = inputs.make_problem(name)
    op = oracle.Problem(prob)
    mp = Problem(prob, device=0, max_chains=max(C, inputs.CONFIGS[name].chains))
    H = inputs.perturbed_heights(prob["H_true"], C, 100 + C, scale=2.0)
    L_d, _ = mp.path_lengths(torch.from_numpy(H).cuda())
    L_d = L_d.cpu().numpy().astype(np.float64)
    L_o, _ = op.path_lengths(H.astype(np.float64))
    err = np.abs(L_d - L_o).max(2) / (1e-5 * L_o.sum(2))
    order = np.argsort(err.ravel())[::-1][:5]
    for flat in order:
        c, q = np.unravel_index(flat, err.shape)
        print(f"chain {c} ray {q}: margin {err[c, q]:.3g}  dev {L_d[c, q]}  ora {L_o[c, q]}")
    c, q = np.unravel_index(order[0], err.shape)
    d = prob["ray_dir"][q]
    o = prob["det_xyz"][prob["ray_det"][q]]
    print("origin", o, "dir", d, "extent", op.ray_extent(q))
    ij_d, si_d, so_d = mp.debug_traversal(q)
    ij_o, si_o, so_o = op.traversal(q)
    print("traversal equal:", np.array_equal(ij_d, ij_o), len(ij_d), len(ij_o))
    Hc = H[c].astype(np.float64)
    n = prob["node_x"].shape[0]
    print("band H0 [%.3f, %.3f] H1 [%.3f, %.3f]" % (Hc[0].min(), Hc[0].max(), Hc[1].min(), Hc[1].max()))
    for k in range(len(ij_o)):
        i, j = ij_o[k]
        z0, z1 = so_o[k] * d[2] if k == 0 else si_o[k] * d[2], so_o[k] * d[2]
        z0 = si_o[k] * d[2]
        hs = [Hc[l].reshape(n, -1)[i:i + 2, j:j + 2].ravel() for l in range(2)]
        flag = ""
        if max(z1, z0) >= min(hs[0].min(), hs[1].min()) - 1 and min(z0, z1) <= max(hs[0].max(), hs[1].max()) + 1:
            flag = " <band>"
        print(f"  {k:3d} ({i:2d},{j:2d}) s [{si_o[k]:.4f}, {so_o[k]:.4f}] dev_s_out {so_d[k]:.4f} z [{z0:.2f}, {z1:.2f}]"
              f" h0 {np.round(hs[0], 2)} h1 {np.round(hs[1], 2)}{flag}")


if __name__ == "__main__":
    main()
