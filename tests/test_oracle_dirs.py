"""Pins of the oracle's real-valued baseline directions (NEXT #2, reading
Q23; orc_detect_dirs / orc_dir_offsets):

* SPEC.md:182-183 worked samples: displacement angle 0 from (50, 20) with
  L = 16 gives x = 42..58 on row 20; displacement pi/4, g = 1 from (10, 10)
  rounds to (11, 11);
* angle 0 with length 1 or 2 is the grid baseline (1, 0) / (2, 0) exactly
  (same samples, W, h, candidates and pairs): equal to the pinned orc_detect
  on random tiny and layered maps, N = infinity and finite N;
* an independent Python implementation (candidates from numpy fp32 edges
  and a binary64 dot product, round-half-away offsets, all ordered pairs of
  each window with the pair test in Fractions for N = infinity, Python's
  stable sort for finite N) equals the oracle on tiny maps at arbitrary
  angles and lengths.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from paper_2408_14050_b200 import scenes

MODES = ["int", "half", "noisy", "uniform"]


def test_spec_scanline_examples(orc):
    dx, dy = orc.dir_offsets(math.pi, 8)           # displacement angle 0
    assert list(50 + dx) == list(range(42, 59)) and (dy == 0).all()
    dx, dy = orc.dir_offsets(math.pi / 4 + math.pi, 1)   # displacement pi/4
    assert (10 + dx[2], 10 + dy[2]) == (11, 11)
    assert (10 + dx[0], 10 + dy[0]) == (9, 9)


@pytest.mark.parametrize("seed", range(6))
def test_angle_zero_is_grid_baseline(orc, seed):
    rng = scenes.SplitMix64(5101, seed)
    for it in range(8):
        H, W = rng.randint(4, 20), rng.randint(4, 20)
        D = scenes.random_tiny_map(rng, H, W, MODES[it % 4])
        N = [0, 0, 2, 8][it % 4]
        a = orc.detect_dirs(D, [(0.0, 1.0), (0.0, 2.0)], neighbors=N)
        b = orc.detect(D, [(1, 0), (2, 0)], neighbors=N)
        assert (a == b).all(), (seed, it)


def _rnd(x):
    return int(math.floor(abs(x) + 0.5)) * (1 if x >= 0 else -1)


def brute_dirs(D, dirs, N=0, t_edge=1.0, t_dist=2.0, t_disp=0.5, max_scan=4096):
    H, W = D.shape
    D = D.astype(np.float32)
    ex = np.zeros_like(D)
    ey = np.zeros_like(D)
    ex[:, :-1] = D[:, 1:] - D[:, :-1]
    ey[:-1, :] = D[1:, :] - D[:-1, :]
    E = np.sqrt((ex * ex) + (ey * ey))               # fp32 throughout
    R = np.float32(D.max() - D.min())
    out = np.zeros((len(dirs), H, W), np.uint8)
    td, tp = Fraction(float(np.float32(t_dist))), Fraction(float(np.float32(t_disp)))
    for vi, (phi, rho) in enumerate(dirs):
        c, s = math.cos(phi), math.sin(phi)
        L = min(max_scan, math.ceil((2.0 * rho) * float(R)))
        h = L // 2
        if h == 0:
            continue
        for y in range(H):
            for x in range(W):
                if not (E[y, x] > np.float32(t_edge) and c * float(ex[y, x]) + s * float(ey[y, x]) > 0.0):
                    continue
                smp = []
                for g in range(-h, h + 1):
                    px, py = x + _rnd(g * -c), y + _rnd(g * -s)
                    if 0 <= px < W and 0 <= py < H:
                        smp.append((g, px, py, D[py, px]))

                def pair(q, p):
                    delta = np.float32(q[3] - p[3])
                    if not Fraction(float(delta)) > tp:
                        return False
                    xr = Fraction(rho * float(delta))      # one binary64 rounding, then exact
                    return abs((q[0] - p[0]) + xr) < td
                if N == 0:
                    for p in smp:
                        if any(pair(q, p) for q in smp if q is not p):
                            out[vi, p[2], p[1]] = 1
                else:
                    w = [Fraction(g) + Fraction(rho * float(v)) for g, _, _, v in smp]
                    wr = [float(g) + rho * float(v) for g, _, _, v in smp]   # binary64 keys
                    order = sorted(range(len(smp)), key=lambda i: (wr[i], i))
                    for r, i in enumerate(order):
                        for d in list(range(-(N // 2), 0)) + list(range(1, N // 2 + 1)):
                            if 0 <= r + d < len(order) and pair(smp[order[r + d]], smp[i]):
                                out[vi, smp[i][2], smp[i][1]] = 1
                                break
    return out


@pytest.mark.parametrize("seed", range(5))
def test_dirs_equal_python_brute(orc, seed):
    rng = scenes.SplitMix64(5102, seed)
    for it in range(4):
        H, W = rng.randint(4, 11), rng.randint(4, 11)
        D = scenes.random_tiny_map(rng, H, W, MODES[it % 4])
        u = rng.uniform(4)
        dirs = [(2 * math.pi * u[0], 1.0), (2 * math.pi * u[1], 0.5 + 2.0 * u[2]), (0.3, 1.0), (2.2, 1.7)]
        for N in (0, 2, 8):
            a = orc.detect_dirs(D, dirs, neighbors=N)
            b = brute_dirs(D, dirs, N)
            assert (a == b).all(), (seed, it, N, dirs)


def test_dirs_validation(orc):
    D = np.zeros((4, 4), np.float32)
    for bad in ([(float("nan"), 1.0)], [(0.0, 0.0)], [(0.0, 9.0)], [(0.0, -1.0)]):
        with pytest.raises(ValueError):
            orc.detect_dirs(D, bad)
    with pytest.raises(ValueError):
        orc.detect_dirs(D, [(0.0, 1.0)], neighbors=3)
