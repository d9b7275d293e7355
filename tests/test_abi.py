"""CPU-side checks of the boundary: libmt.so builds for sm_100a, loads, and
exports every symbol include/mt.h declares (no compute calls without a GPU)."""
import ctypes as ct
import os
import re
import subprocess

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
