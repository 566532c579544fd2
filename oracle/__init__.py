"""ctypes front end of the CPU ORACLE (oracle/occ_oracle.c, oracle/brute.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs.  The product path
(``paper_2408_14050_b200``) never imports this package.

The shared library is compiled with ``-O2 -ffp-contract=off -fno-fast-math``
so every fp32 operation is a single IEEE round-to-nearest-even operation
(fp recipe).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = [os.path.join(_HERE, "occ_oracle.c"), os.path.join(_HERE, "brute.c")]
CFLAGS = ["-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-ffp-contract=off", "-fno-fast-math",
          "-fPIC", "-shared", "-Wall", "-Wextra"]

OK, ERR_INVALID_ARG, ERR_NONFINITE, ERR_UNSUPPORTED = 0, -1, -4, -5
DEFAULTS = dict(t_edge=1.0, t_dist=2.0, t_disp=0.5, max_scan=4096)


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (gcc).  Returns its path."""
    newest = max(os.path.getmtime(s) for s in _SRCS + [os.path.join(_HERE, "occ_oracle.h")])
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", *CFLAGS, "-o", _SO, *_SRCS, "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        f32p = ctypes.POINTER(ctypes.c_float)
        i32p = ctypes.POINTER(ctypes.c_int32)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        f64p = ctypes.POINTER(ctypes.c_double)
        i32, f32 = ctypes.c_int32, ctypes.c_float
        sig = {
            "orc_validate": (ctypes.c_int, [i32, i32, i32p, i32, f32, f32, f32, i32]),
            "orc_stats": (ctypes.c_int64, [f32p, i32, i32, f32p, f32p]),
            "orc_edges": (None, [f32p, i32, i32, f32p, f32p, f32p]),
            "orc_candidates": (ctypes.c_int64, [f32p, f32p, f32p, i32, i32, i32, i32, f32, u8p]),
            "orc_angle_predicate": (ctypes.c_int, [f32, f32, i32, i32]),
            "orc_scan_length": (i32, [f32, f32, i32, i32]),
            "orc_scanline": (i32, [f32p, i32, i32, i32, i32, i32, i32, i32, i32p, i32p, i32p, f32p]),
            "orc_sort": (None, [f64p, i32, i32p]),
            "orc_pair": (ctypes.c_int, [f32, f32, i32, i32, f32, f32]),
            "orc_count": (None, [i32p, f32p, f64p, i32p, i32, i32, f32, f32, ctypes.c_double, i32p]),
            "orc_detect": (ctypes.c_int, [f32p, i32, i32, i32p, i32, f32, f32, f32, i32, u8p, i32p]),
            "bf1_detect": (ctypes.c_int, [f32p, i32, i32, i32p, i32, f32, f32, f32, i32, u8p]),
            "bf2_zbuffer": (ctypes.c_int, [f32p, i32, i32, i32, i32, f32, u8p]),
            "orc_fuse_median": (ctypes.c_int, [f32p, i32, ctypes.c_int64, f32p]),
            "orc_count_n": (None, [i32p, f32p, i32p, i32, i32, f32, f32, i32, i32p]),
            "orc_detect_dirs": (ctypes.c_int, [f32p, i32, i32, f64p, f64p, i32, f32, f32, f32, i32, i32, u8p, i32p]),
            "orc_dir_offsets": (ctypes.c_int, [ctypes.c_double, i32, i32p, i32p]),
            "orc_detect_range": (ctypes.c_int, [f32p, i32, i32, i32p, i32, f32, f32, f32, i32, i32, f32, f32,
                                                u8p, i32p]),
            "orc_detect_n": (ctypes.c_int, [f32p, i32, i32, i32p, i32, f32, f32, f32, i32, i32, u8p, i32p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _baselines(views: Sequence[Tuple[int, int]]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(views, dtype=np.int32).reshape(-1, 2))


def detect(D: np.ndarray, views: Sequence[Tuple[int, int]], t_edge: float = 1.0,
           t_dist: float = 2.0, t_disp: float = 0.5, max_scan: int = 4096,
           return_info: bool = False, neighbors: int = 0):
    """Oracle masks uint8 [V, H, W] for one fp32 [H, W] map; raises on error codes
    other than NONFINITE (which returns zero masks and rc)."""
    D = np.ascontiguousarray(D, dtype=np.float32)
    H, W = D.shape
    b = _baselines(views)
    V = b.shape[0]
    masks = np.zeros((V, H, W), dtype=np.uint8)
    info = np.zeros((V, 4), dtype=np.int32)
    rc = lib().orc_detect_n(_p(D, ctypes.c_float), H, W, _p(b, ctypes.c_int32), V,
                            t_edge, t_dist, t_disp, max_scan, int(neighbors),
                            _p(masks, ctypes.c_uint8), _p(info, ctypes.c_int32))
    if rc not in (OK, ERR_NONFINITE):
        raise ValueError(f"orc_detect rc={rc}")
    if return_info:
        return masks, info, rc
    return masks


def detect_rc(D: np.ndarray, views, **kw) -> int:
    return detect(D, views, return_info=True, **kw)[2]


def validate(H, W, views, t_edge=1.0, t_dist=2.0, t_disp=0.5, max_scan=4096) -> int:
    b = _baselines(views) if len(views) else np.zeros((0, 2), np.int32)
    ptr = _p(b, ctypes.c_int32) if len(views) else None
    return lib().orc_validate(H, W, ptr, len(views), t_edge, t_dist, t_disp, max_scan)


def bf1(D: np.ndarray, views, t_edge=1.0, t_dist=2.0, t_disp=0.5, max_scan=4096) -> np.ndarray:
    D = np.ascontiguousarray(D, dtype=np.float32)
    H, W = D.shape
    b = _baselines(views)
    masks = np.zeros((b.shape[0], H, W), dtype=np.uint8)
    rc = lib().bf1_detect(_p(D, ctypes.c_float), H, W, _p(b, ctypes.c_int32), b.shape[0],
                          t_edge, t_dist, t_disp, max_scan, _p(masks, ctypes.c_uint8))
    if rc != OK:
        raise ValueError(f"bf1 rc={rc}")
    return masks


def bf2(D: np.ndarray, b: Tuple[int, int], t_disp: float = 0.5) -> np.ndarray:
    D = np.ascontiguousarray(D, dtype=np.float32)
    H, W = D.shape
    m = np.zeros((H, W), dtype=np.uint8)
    rc = lib().bf2_zbuffer(_p(D, ctypes.c_float), H, W, b[0], b[1], t_disp, _p(m, ctypes.c_uint8))
    if rc != OK:
        raise ValueError(f"bf2 rc={rc}")
    return m


def stats(D: np.ndarray):
    D = np.ascontiguousarray(D, dtype=np.float32)
    lo, hi = ctypes.c_float(), ctypes.c_float()
    bad = lib().orc_stats(_p(D, ctypes.c_float), D.shape[0], D.shape[1], ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value, int(bad)


def edges(D: np.ndarray):
    D = np.ascontiguousarray(D, dtype=np.float32)
    H, W = D.shape
    Ex, Ey, E = (np.zeros((H, W), np.float32) for _ in range(3))
    lib().orc_edges(_p(D, ctypes.c_float), H, W, _p(Ex, ctypes.c_float), _p(Ey, ctypes.c_float),
                    _p(E, ctypes.c_float))
    return Ex, Ey, E


def candidates(D: np.ndarray, b: Tuple[int, int], t_edge: float = 1.0) -> np.ndarray:
    Ex, Ey, E = edges(D)
    H, W = Ex.shape
    c = np.zeros((H, W), np.uint8)
    lib().orc_candidates(_p(Ex, ctypes.c_float), _p(Ey, ctypes.c_float), _p(E, ctypes.c_float),
                         H, W, b[0], b[1], t_edge, _p(c, ctypes.c_uint8))
    return c


def angle_predicate(ex: float, ey: float, b: Tuple[int, int]) -> int:
    return lib().orc_angle_predicate(ex, ey, b[0], b[1])


def scan_length(dmin: float, dmax: float, s: int = 1, max_scan: int = 4096) -> int:
    return lib().orc_scan_length(dmin, dmax, s, max_scan)


def scanline(D: np.ndarray, b, c: Tuple[int, int], h: int):
    D = np.ascontiguousarray(D, dtype=np.float32)
    H, W = D.shape
    n = 2 * h + 1
    g, xs, ys = (np.zeros(n, np.int32) for _ in range(3))
    v = np.zeros(n, np.float32)
    k = lib().orc_scanline(_p(D, ctypes.c_float), H, W, b[0], b[1], c[0], c[1], h,
                           _p(g, ctypes.c_int32), _p(xs, ctypes.c_int32), _p(ys, ctypes.c_int32),
                           _p(v, ctypes.c_float))
    return g[:k], xs[:k], ys[:k], v[:k]


def sort(w) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.float64)
    idx = np.zeros(len(w), np.int32)
    lib().orc_sort(_p(w, ctypes.c_double), len(w), _p(idx, ctypes.c_int32))
    return idx


def pair(vq: float, vp: float, dk: int, s: int = 1, t_dist: float = 2.0, t_disp: float = 0.5) -> int:
    return lib().orc_pair(vq, vp, dk, s, t_dist, t_disp)


def count(g, v, w, idx, s=1, t_dist=2.0, t_disp=0.5, eps=1e-6) -> np.ndarray:
    g = np.ascontiguousarray(g, np.int32)
    v = np.ascontiguousarray(v, np.float32)
    w = np.ascontiguousarray(w, np.float64)
    idx = np.ascontiguousarray(idx, np.int32)
    O = np.zeros(len(g), np.int32)
    lib().orc_count(_p(g, ctypes.c_int32), _p(v, ctypes.c_float), _p(w, ctypes.c_double),
                    _p(idx, ctypes.c_int32), len(g), s, t_dist, t_disp, eps, _p(O, ctypes.c_int32))
    return O


def fuse_median(stack: np.ndarray) -> np.ndarray:
    """Pixel-wise median of K fp32 estimates:
    stack [K, ...] -> [...]; even K: fl32(fl32(a + b) * 0.5) of the middle pair;
    NaN where any estimate is non-finite."""
    st = np.ascontiguousarray(stack, dtype=np.float32)
    K = st.shape[0]
    n = int(np.prod(st.shape[1:])) if st.ndim > 1 else 1
    out = np.empty(st.shape[1:], dtype=np.float32)
    rc = lib().orc_fuse_median(_p(st, ctypes.c_float), K, n, _p(out, ctypes.c_float))
    if rc != OK:
        raise ValueError(f"orc_fuse_median rc={rc}")
    return out


def count_n(g, v, idx, N, s=1, t_dist=2.0, t_disp=0.5) -> np.ndarray:
    """O10 with a finite neighbour count N over a sorted line (orc_count_n)."""
    g = np.ascontiguousarray(g, np.int32)
    v = np.ascontiguousarray(v, np.float32)
    idx = np.ascontiguousarray(idx, np.int32)
    O = np.zeros(len(g), np.int32)
    lib().orc_count_n(_p(g, ctypes.c_int32), _p(v, ctypes.c_float), _p(idx, ctypes.c_int32), len(g), s,
                      t_dist, t_disp, int(N), _p(O, ctypes.c_int32))
    return O


def detect_range(D: np.ndarray, views, dmin: float, dmax: float, t_edge: float = 1.0, t_dist: float = 2.0,
                 t_disp: float = 0.5, max_scan: int = 4096, neighbors: int = 0) -> np.ndarray:
    """orc_detect_range: masks of D with Eq. 3's min / max imposed (a band of a
    larger frame whose statistics are dmin, dmax)."""
    D = np.ascontiguousarray(D, dtype=np.float32)
    H, W = D.shape
    b = _baselines(views)
    masks = np.zeros((b.shape[0], H, W), dtype=np.uint8)
    info = np.zeros((b.shape[0], 4), dtype=np.int32)
    rc = lib().orc_detect_range(_p(D, ctypes.c_float), H, W, _p(b, ctypes.c_int32), b.shape[0], t_edge, t_dist,
                                t_disp, max_scan, int(neighbors), float(dmin), float(dmax),
                                _p(masks, ctypes.c_uint8), _p(info, ctypes.c_int32))
    if rc != OK:
        raise ValueError(f"orc_detect_range rc={rc}")
    return masks


def detect_dirs(D: np.ndarray, dirs, t_edge: float = 1.0, t_dist: float = 2.0, t_disp: float = 0.5,
                max_scan: int = 4096, neighbors: int = 0, return_info: bool = False):
    """NEXT #2 (reading Q23): dirs = [(baseline_angle_rad, baseline_length), ...]."""
    D = np.ascontiguousarray(D, dtype=np.float32)
    H, W = D.shape
    phi = np.ascontiguousarray([float(a) for a, _ in dirs], np.float64)
    rho = np.ascontiguousarray([float(r) for _, r in dirs], np.float64)
    V = len(dirs)
    masks = np.zeros((V, H, W), dtype=np.uint8)
    info = np.zeros((V, 4), dtype=np.int32)
    rc = lib().orc_detect_dirs(_p(D, ctypes.c_float), H, W, _p(phi, ctypes.c_double), _p(rho, ctypes.c_double), V,
                               t_edge, t_dist, t_disp, max_scan, int(neighbors), _p(masks, ctypes.c_uint8),
                               _p(info, ctypes.c_int32))
    if rc not in (OK, ERR_NONFINITE):
        raise ValueError(f"orc_detect_dirs rc={rc}")
    return (masks, info, rc) if return_info else masks


def dir_offsets(phi: float, h: int):
    dx = np.zeros(2 * h + 1, np.int32)
    dy = np.zeros(2 * h + 1, np.int32)
    rc = lib().orc_dir_offsets(float(phi), int(h), _p(dx, ctypes.c_int32), _p(dy, ctypes.c_int32))
    if rc != OK:
        raise ValueError(f"orc_dir_offsets rc={rc}")
    return dx, dy
