"""C ABI checks that need no GPU: the library loads, exports every function
include/occ.h declares, and rejects invalid arguments before touching CUDA
(occ_create validates first)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def occ():
    from paper_2408_14050_b200 import build
    build.build()
    from paper_2408_14050_b200 import occ as m
    return m


def header_functions():
    src = open(os.path.join(ROOT, "include", "occ.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(occ_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(occ):
    funcs = header_functions()
    assert len(funcs) >= 10
    out = subprocess.run(["nm", "-D", "--defined-only", occ.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (occ_\w+)", out))
    missing = [f for f in funcs if f not in exported]
    assert not missing, missing
    L = occ.lib()
    for f in funcs:
        assert getattr(L, f) is not None
    assert sorted(occ.EXPORTS) == funcs


def test_no_torch_or_oracle_in_library(occ):
    out = subprocess.run(["nm", "-D", occ.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out and "bf1_" not in out and "torch" not in out
    ldd = subprocess.run(["ldd", occ.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in ldd and "oracle" not in ldd


def test_defaults_and_strings(occ):
    p = occ.default_params()
    assert (p.t_edge, p.t_dist, p.t_disp, p.max_scan) == (1.0, 2.0, 0.5, 4096)
    assert occ.lib().occ_version() == 10000
    for code in (0, -1, -2, -3, -4, -5):
        assert occ.strerror(code)
    assert occ.strerror(-4) == "non-finite disparity in frame"


@pytest.mark.parametrize("H,W,views,kw,expect", [
    (1, 8, [(1, 0)], {}, -1),          # SPEC.md:113 map smaller than 2x2
    (8, 1, [(1, 0)], {}, -1),
    (8, 8, [], {}, -1),                # no views
    (8, 8, [(0, 0)], {}, -1),          # b = (0, 0)
    (8, 8, [(9, 1)], {}, -5),          # |b| > 8 unsupported
    (8, 8, [(1, 0)], {"t_edge": 0.0}, -1),
    (8, 8, [(1, 0)], {"t_edge": float("nan")}, -1),
    (8, 8, [(1, 0)], {"t_dist": 0.0}, -1),
    (8, 8, [(1, 0)], {"t_dist": 1e6}, -1),
    (8, 8, [(1, 0)], {"t_disp": -0.5}, -1),
    (8, 8, [(1, 0)], {"max_scan": 0}, -1),
    (8, 8, [(1, 0)], {"max_batch": 0}, -1),
    (40000, 8, [(1, 0)], {}, -1),
])
def test_create_validation(occ, H, W, views, kw, expect):
    p = occ.default_params()
    for k in ("t_edge", "t_dist", "t_disp", "max_scan"):
        if k in kw:
            setattr(p, k, kw[k])
    rc, h = occ.create_raw(H, W, views, p, kw.get("max_batch", 1))
    assert rc == expect and h is None


def test_null_out_pointer(occ):
    L = occ.lib()
    arr = (occ.occ_baseline * 1)(occ.occ_baseline(1, 0))
    assert L.occ_create(8, 8, arr, 1, None, 1, None) == -1
    assert L.occ_detect(None, None, None, 1, None) == -1
    assert L.occ_destroy(None) == -1
    assert L.occ_set_path(None, 0) == -1
    assert L.occ_last_launches(None) == -1
