"""CPU-side checks of the boundary: libmt.so builds for sm_100a, loads, and
exports every symbol include/mt.h declares (no compute calls without a GPU)."""
import ctypes as ct
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mt_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def so_path():
    from paper_2603_28907_b200 import build
    return build.build()


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for s in ("mt_problem_create", "mt_logpost_grad", "mt_leapfrog", "mt_problem_destroy",
              "mt_hmc_step", "mt_draw_momenta", "mt_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(so_path):
    L = ct.CDLL(so_path)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    from paper_2603_28907_b200 import _lib
    assert set(_lib.EXPORTS) == set(declared_symbols())


def test_library_is_sm100a_cubin(so_path):
    out = subprocess.run(["cuobjdump", "--list-elf", so_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_and_invalid_arguments_fail_loudly(so_path):
    L = ct.CDLL(so_path)
    L.mt_problem_create.argtypes = [ct.c_void_p, ct.c_void_p]
    L.mt_last_error.restype = ct.c_char_p
    assert L.mt_problem_create(None, None) == 1
    assert b"out is NULL" in L.mt_last_error()
    h = ct.c_void_p()
    assert L.mt_problem_create(None, ct.byref(h)) == 1
    assert L.mt_problem_destroy(None) == 0


def test_product_path_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2603_28907_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle.c" not in txt and "liboracle" not in txt, f


def test_widening_entry_points_validate_before_touching_the_device(so_path, problems):
    """f2/f3 entry points reject bad arguments with MT_EINVAL (no GPU needed)."""
    from paper_2603_28907_b200 import inputs
    from paper_2603_28907_b200._lib import _Desc
    L = ct.CDLL(so_path)
    L.mt_last_error.restype = ct.c_char_p
    L.mt_voxel_model.argtypes = [ct.c_void_p, ct.c_int32, ct.c_float, ct.c_float, ct.c_void_p]
    L.mt_voxel_info.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p]
    L.mt_voxel_counters.argtypes = [ct.c_void_p, ct.c_void_p]
    L.mt_measure_l2_gather.argtypes = [ct.c_int32, ct.c_int64, ct.c_void_p]
    assert L.mt_voxel_model(None, 60, 1.0, 1e-3, None) == 1
    assert b"problem is NULL" in L.mt_last_error()
    assert L.mt_voxel_info(None, None, None, None) == 1
    assert L.mt_voxel_counters(None, None) == 1
    v = ct.c_double()
    assert L.mt_measure_l2_gather(0, 1024, ct.byref(v)) == 1
    # noncentred without sample_r: a descriptor error, found before any device query
    prob = problems("tiny")
    keep = {k: np.ascontiguousarray(prob[k], dt) for k, dt in
            (("node_x", np.float32), ("node_y", np.float32), ("det_xyz", np.float32), ("ray_det", np.int32),
             ("ray_dir", np.float32), ("ray_w", np.float32), ("counts", np.int32))}
    d = _Desc()
    d.n_x = d.n_y = len(keep["node_x"])
    d.node_x, d.node_y = keep["node_x"].ctypes.data, keep["node_y"].ctypes.data
    d.z_top, d.rho_muck, d.rho_air, d.rho_rock, d.rho_ext, d.att_len = 300.0, 1.9, 0.0012, 2.65, 2.65, 250.0
    d.car_r[0] = d.car_r[1] = 0.95
    d.n_det, d.det_xyz = len(keep["det_xyz"]), keep["det_xyz"].ctypes.data
    d.n_rays = len(keep["ray_det"])
    d.ray_det, d.ray_dir = keep["ray_det"].ctypes.data, keep["ray_dir"].ctypes.data
    d.ray_w, d.counts = keep["ray_w"].ctypes.data, keep["counts"].ctypes.data
    d.ray_lo, d.ray_hi, d.max_chains = 0, d.n_rays, 4
    d.sample_r, d.noncentred = 0, 1
    L.mt_problem_create.argtypes = [ct.c_void_p, ct.c_void_p]
    h = ct.c_void_p()
    assert L.mt_problem_create(ct.byref(d), ct.byref(h)) == 1
    assert b"noncentred requires sample_r" in L.mt_last_error()
    assert inputs.CONFIGS["tiny"].n == d.n_x
