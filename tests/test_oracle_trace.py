"""Oracle pins: traversal, exact path lengths and opacity.

Pins: exact rational brute force over all cells (fractions.Fraction), closed
forms for flat / planar / vertical cases, fine-step midpoint marching with a
library bilinear interpolator (scipy RegularGridInterpolator), and the sign
/ invariance properties the paper's unit map implies.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest
from scipy.interpolate import RegularGridInterpolator

import oracle
from paper_2603_28907_b200 import inputs


def custom_problem(base, det_xyz, dirs, counts=None, w=None, **over):
    p = dict(base)
    p["det_xyz"] = np.asarray(det_xyz, np.float32).reshape(-1, 3)
    dirs = np.asarray(dirs, np.float64).reshape(-1, 3)
    dirs = dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    p["ray_dir"] = dirs.astype(np.float32)
    R = len(dirs)
    p["ray_det"] = np.zeros(R, np.int32) if len(p["det_xyz"]) == 1 else np.arange(R, dtype=np.int32)
    p["ray_w"] = np.full(R, 1000.0, np.float32) if w is None else np.asarray(w, np.float32)
    p["counts"] = np.full(R, 900, np.int32) if counts is None else np.asarray(counts, np.int32)
    p.update(over)
    return p


def brute_cells(X, Y, ztop, o, d):
    """All cells whose exact parameter interval inside [0, s_exit] has positive length."""
    X = [Fr(float(v)) for v in X]
    Y = [Fr(float(v)) for v in Y]
    o = [Fr(float(v)) for v in o]
    d = [Fr(float(v)) for v in d]
    zt = Fr(float(ztop))

    def slab(lo, hi, oo, dd):
        if dd == 0:
            # a ray lying on a grid line belongs to the cell above the line (R16)
            return (Fr(-10 ** 9), Fr(10 ** 9)) if lo <= oo < hi else None
        a, b = (lo - oo) / dd, (hi - oo) / dd
        return (min(a, b), max(a, b))
    sx = slab(X[0], X[-1], o[0], d[0])
    sy = slab(Y[0], Y[-1], o[1], d[1])
    s_exit = min(sx[1], sy[1], (zt - o[2]) / d[2])
    cells = []
    for i in range(len(X) - 1):
        ix = slab(X[i], X[i + 1], o[0], d[0])
        if ix is None:
            continue
        for j in range(len(Y) - 1):
            iy = slab(Y[j], Y[j + 1], o[1], d[1])
            if iy is None:
                continue
            a = max(ix[0], iy[0], Fr(0))
            b = min(ix[1], iy[1], s_exit)
            if b > a:
                cells.append((a, b, i, j))
    cells.sort()
    return cells, s_exit


def check_traversal(op, q):
    prob = op.prob
    o = prob["det_xyz"][prob["ray_det"][q]]
    d = prob["ray_dir"][q]
    ij, si, so = op.traversal(q)
    cells, s_exit = brute_cells(prob["node_x"], prob["node_y"], prob["z_top"], o, d)
    assert [tuple(c[2:]) for c in cells] == [tuple(v) for v in ij], q
    assert np.allclose(si, [float(c[0]) for c in cells], rtol=1e-13, atol=1e-12)
    assert np.allclose(so, [float(c[1]) for c in cells], rtol=1e-13, atol=1e-12)
    assert np.all(so > si) and np.all(si[1:] == so[:-1])
    assert abs(np.sum(so - si) - float(s_exit)) <= 1e-12 * float(s_exit)
    se, _ = op.ray_extent(q)
    assert se == pytest.approx(float(s_exit), rel=1e-15)


def test_traversal_tiny_all_rays(oracle_problem):
    op = oracle_problem("tiny")
    for q in range(op.R):
        check_traversal(op, q)


def test_traversal_small_sample(oracle_problem):
    op = oracle_problem("small")
    for q in np.random.default_rng(1).choice(op.R, 200, replace=False):
        check_traversal(op, int(q))


def test_traversal_special_rays(problems):
    base = problems("tiny")
    # uniform 12.5 m grid so rays through vertices are exact
    X = (np.arange(9) * 12.5).astype(np.float32)
    b = dict(base, node_x=X, node_y=X.copy())
    dets = [(25.0, 37.5, 0.0), (50.0, 50.0, 0.0), (31.25, 60.0, 0.0), (0.5, 0.5, 0.0), (99.5, 50.0, 0.0)]
    dirs = [(1, 1, 1), (-1, 1, 2), (1, 0, 1), (0, -1, 1), (0, 0, 1), (1, 1, 0.05), (-1, 0, 0.3),
            (0.3, -1, 0.2)]
    for o in dets:
        p = custom_problem(b, [o], dirs)
        op = oracle.Problem(p)
        for q in range(len(dirs)):
            check_traversal(op, q)
    # axis-parallel ray visits one row of cells, in order
    p = custom_problem(b, [(30.0, 40.0, 0.0)], [(1, 0, 0.01)])
    ij, _, _ = oracle.Problem(p).traversal(0)
    assert [tuple(v) for v in ij] == [(k, 3) for k in range(2, 8)]
    # diagonal through vertices skips the diagonal neighbours
    p = custom_problem(b, [(25.0, 37.5, 0.0)], [(1, 1, 0.02)])
    ij, _, _ = oracle.Problem(p).traversal(0)
    assert [tuple(v) for v in ij] == [(2 + k, 3 + k) for k in range(5)]


# --------------------------------------------------------------------------
# path lengths
# --------------------------------------------------------------------------

def flat_heights(n, c0, c1):
    return np.stack([np.full((n, n), c0), np.full((n, n), c1)])[None]


def test_flat_surfaces_closed_form(oracle_problem):
    op = oracle_problem("small")
    c0, c1 = 120.0, 170.0
    L, O = op.path_lengths(flat_heights(op.nx, c0, c1))
    d = op.prob["ray_dir"].astype(np.float64)
    se = np.array([op.ray_extent(q)[0] for q in range(op.R)])
    B0 = np.minimum(c0 / d[:, 2], se)
    B1 = np.minimum(c1 / d[:, 2], se)
    assert np.allclose(L[0, :, 0], B0, rtol=1e-12)
    assert np.allclose(L[0, :, 1], B1 - B0, rtol=1e-12, atol=1e-9)
    assert np.allclose(L[0].sum(1), se, rtol=1e-12)
    top = np.isclose(se, op.z_top / d[:, 2], rtol=1e-15)
    assert top.sum() > 100
    # thickness / cos(zenith) exactly for top-exit rays
    assert np.allclose(L[0, top, 1], (c1 - c0) / d[top, 2], rtol=1e-12)


def test_planar_surfaces_closed_form(oracle_problem):
    op = oracle_problem("small")
    X = op.prob["node_x"].astype(np.float64)
    xx, yy = np.meshgrid(X, X, indexing="ij")
    al, be, ga = 140.0, 0.08, -0.05
    H = np.stack([al + be * xx + ga * yy, al + 30 + be * xx + ga * yy])[None]
    L, _ = op.path_lengths(H)
    o = op.prob["det_xyz"][op.prob["ray_det"]].astype(np.float64)
    d = op.prob["ray_dir"].astype(np.float64)
    se = np.array([op.ray_extent(q)[0] for q in range(op.R)])
    for l, a in ((0, al), (1, al + 30)):
        s_star = (a + be * o[:, 0] + ga * o[:, 1] - o[:, 2]) / (d[:, 2] - be * d[:, 0] - ga * d[:, 1])
        B = np.where((s_star > 0) & (s_star < se), s_star, se)
        Bo = L[0, :, 0] if l == 0 else L[0, :, 0] + L[0, :, 1]
        assert np.allclose(Bo, B, rtol=1e-11)


def test_vertical_ray_bilinear_and_gradient(problems):
    base = problems("small")
    rng = np.random.default_rng(5)
    H = inputs.perturbed_heights(base["H_true"], 1, 11, scale=3.0).astype(np.float64)
    dets = [(37.3, 81.9, 0.0), (150.1, 12.7, 0.0), (100.0 + 1 / 4096, 133.3, 0.0)]
    X = base["node_x"].astype(np.float64)
    for det in dets:
        det = inputs.quantize(det)
        p = custom_problem(base, [det], [(0, 0, 1)])
        op = oracle.Problem(p)
        L, O = op.path_lengths(H)
        for l in (0, 1):
            f = RegularGridInterpolator((X, X), H[0, l], method="linear")
            ref = f([det[:2]])[0]
            B = L[0, 0, 0] if l == 0 else L[0, 0, 0] + L[0, 0, 1]
            assert B == pytest.approx(ref, rel=1e-13)
        # ∂B/∂h_node = bilinear weight φ_node; read through dll/dH = (λ-C)/Λ·∂O/∂B_l·∂B/∂h
        out = op.loglik_grad_H(H)
        lam = p["ray_w"][0] * np.exp(-O[0, 0] / p["att_len"])
        dldO = (lam - p["counts"][0]) / p["att_len"]
        for l, k in ((0, p["rho_muck"] - p["rho_air"]), (1, p["rho_air"] - p["rho_rock"])):
            phi = out["dldH"][0, l] / (dldO * k)
            ref = np.zeros_like(phi)
            for i in range(len(X)):
                e = np.zeros(len(X))
                e[i] = 1.0
                for j in range(len(X)):
                    e2 = np.zeros(len(X))
                    e2[j] = 1.0
                    w = RegularGridInterpolator((X, X), np.outer(e, e2), method="linear")([det[:2]])[0]
                    ref[i, j] = w
            assert np.allclose(phi, ref, atol=1e-12)


def test_bruteforce_marching_tiny(problems):
    base = problems("tiny")
    op = oracle.Problem(base)
    H = inputs.perturbed_heights(base["H_true"], 2, 3, scale=4.0).astype(np.float64)
    L, _ = op.path_lengths(H)
    X = base["node_x"].astype(np.float64)
    ds = 2e-3
    for c in range(2):
        fs = [RegularGridInterpolator((X, X), H[c, l], method="linear") for l in (0, 1)]
        for q in range(0, op.R, 5):
            o = base["det_xyz"][0].astype(np.float64)
            d = base["ray_dir"][q].astype(np.float64)
            se, _ = op.ray_extent(q)
            n = int(np.floor(se / ds))
            s = (np.arange(n) + 0.5) * ds
            pts = o[None, :] + s[:, None] * d[None, :]
            rem = se - n * ds
            for l in (0, 1):
                below = pts[:, 2] < fs[l](pts[:, :2])
                Bbf = ds * below.sum()
                Bo = L[c, q, 0] if l == 0 else L[c, q, 0] + L[c, q, 1]
                ncross = np.count_nonzero(np.diff(below.astype(int)))
                assert abs(Bo - Bbf) <= (ncross + 1) * ds + rem + 1e-9, (c, q, l)


def test_misses_and_sums(oracle_problem):
    op = oracle_problem("small")
    H = op.prob["H_true"][None]
    L, O = op.path_lengths(H)
    d = op.prob["ray_dir"].astype(np.float64)
    se = np.array([op.ray_extent(q)[0] for q in range(op.R)])
    miss = se * d[:, 2] < H[0, 0].min()           # leaves the box below every surface
    assert miss.sum() > 10
    assert np.allclose(L[0, miss, 1], 0, atol=1e-12 * 400) and np.allclose(L[0, miss, 2], 0, atol=1e-12 * 400)
    assert np.allclose(L[0].sum(1), se, rtol=1e-12)
    assert np.all(L[0] >= -1e-9)


def test_opacity_invariants(problems):
    base = problems("tiny")
    eq = dict(base, rho_muck=2.0, rho_air=2.0, rho_rock=2.0, rho_ext=2.0)
    op = oracle.Problem(eq)
    H1 = inputs.perturbed_heights(base["H_true"], 3, 4, scale=5.0)
    _, O = op.path_lengths(H1)
    ext = np.array([sum(op.ray_extent(q)) for q in range(op.R)])
    assert np.allclose(O, 2.0 * ext[None], rtol=1e-12)
    # monotone in each node: raising H0 never lowers O, raising H1 never raises O
    op = oracle.Problem(base)
    H = inputs.perturbed_heights(base["H_true"], 1, 5, scale=2.0).astype(np.float64)
    _, O0 = op.path_lengths(H)
    rng = np.random.default_rng(9)
    for _ in range(10):
        i, j = rng.integers(0, op.nx, 2)
        Hp = H.copy()
        Hp[0, 0, i, j] += 3.0
        _, Op = op.path_lengths(Hp)
        assert np.all(Op >= O0 - 1e-9)
        Hp = H.copy()
        Hp[0, 1, i, j] += 3.0
        _, Op = op.path_lengths(Hp)
        assert np.all(Op <= O0 + 1e-9)


def test_work_counters_vs_brute_force(problems, oracle_problem):
    """The oracle's instrumentation, which sets the roofline's
    algorithmic work (tools/count_work.py), against counts recomputed here from their
    definitions: in-box cells (the traversal), band cells (cell z-range meets
    (min H0, max H1)), unresolved surface-cells (z-range meets the cell's corner range)
    and crossings (sign changes of g = h - z sampled every 2.5 mm along each ray)."""
    name = "tiny"
    prob, op = problems(name), oracle_problem(name)
    x = inputs.chain_states(prob["x_true"], 2, inputs.CONFIGS[name].seed, scale=0.3)
    H = np.stack([op.heights(xc.astype(np.float64))[0] for xc in x])
    cnt = op.logpost_grad(x.astype(np.float64))["counters"]
    off, ij, so = op.traversal_all()
    si = np.concatenate([[0.0], so[:-1]])
    si[off[:-1]] = 0.0                                   # each ray's first cell starts at s = 0
    ray = np.repeat(np.arange(op.R), np.diff(off))
    dz = np.asarray(prob["ray_dir"], np.float64)[ray, 2]
    za, zb = si * dz, so * dz
    n_inbox = n_band = n_unres = n_cross = 0
    X = np.asarray(prob["node_x"], np.float64)
    Y = np.asarray(prob["node_y"], np.float64)
    o = np.asarray(prob["det_xyz"], np.float64)[np.asarray(prob["ray_det"])]
    d = np.asarray(prob["ray_dir"], np.float64)
    for c in range(2):
        n_inbox += len(ij)
        n_band += int(np.sum((zb > H[c, 0].min()) & (za < H[c, 1].max())))
        for l in range(2):
            h = H[c, l]
            c4 = np.stack([h[ij[:, 0], ij[:, 1]], h[ij[:, 0] + 1, ij[:, 1]], h[ij[:, 0], ij[:, 1] + 1],
                           h[ij[:, 0] + 1, ij[:, 1] + 1]])
            n_unres += int(np.sum(~((zb <= c4.min(0)) | (za >= c4.max(0)))))
            interp = RegularGridInterpolator((X, Y), h)
            for q in range(op.R):
                s_exit, _ = op.ray_extent(q)
                s = np.arange(0.00125, s_exit, 0.0025)
                p = o[q][None, :] + s[:, None] * d[q][None, :]
                g = interp(np.clip(p[:, :2], [X[0], Y[0]], [X[-1], Y[-1]])) - p[:, 2]
                n_cross += int(np.sum(np.sign(g[1:]) != np.sign(g[:-1])))
    assert cnt[0] == n_inbox and cnt[1] == n_band and cnt[2] == n_unres
    assert cnt[3] == n_cross, (cnt, n_cross)


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_bulk_traversal_equals_the_per_ray_traversal(problems, oracle_problem, name):
    """or_traversal_all (the bulk CSR the exhaustive GPU test compares against) is the
    per-ray traversal (itself pinned by exact rational brute force above), ray by ray:
    same cells in the same order, same exit parameters."""
    op = oracle_problem(name)
    off, ij, so = op.traversal_all()
    assert off[0] == 0 and np.all(np.diff(off) >= 0)
    for q in range(0, op.R, 1 if op.R <= 256 else 53):
        ij_q, _, so_q = op.traversal(q)
        assert np.array_equal(ij[off[q]:off[q + 1]], ij_q), q
        assert np.array_equal(so[off[q]:off[q + 1]], so_q), q
