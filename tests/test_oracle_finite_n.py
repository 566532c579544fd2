"""Pins of the oracle's finite-N count (orc_count_n /
orc_detect_n): Eq. 5 of PAPER.md:131-142 taken literally, each sorted entry
compared with its N nearest sorted neighbours (d in {-N/2..-1, 1..N/2},
SPEC.md:197; N = 8 is SPEC.md:155's default).

* the SPEC.md:201 worked example at N = 8, and the same line at N = 2 / 4
  worked by hand (tests/golden/spec_examples.json "count_n");
* N >= 2 (2h + 1) reaches every entry of the line, so the masks equal the
  N = infinity oracle (pinned itself against brute.c's BF1);
* masks grow monotonically with N (the neighbour sets are nested);
* an independent Python brute force on tiny maps: exact rational warped
  coordinates, Python's stable sort on (w, scan index), the exact pair test
  in Fractions -- sharing only the separately pinned window samples
  (orc_scanline) and candidate map (orc_candidates) with the oracle;
* argument validation (odd or N < 2 rejected; N = 0 = infinity).
"""
import json
import pathlib
from fractions import Fraction

import numpy as np
import pytest

from paper_2408_14050_b200 import scenes

GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "spec_examples.json").read_text())


def _line_sort(g, v, s):
    w = [Fraction(int(gi)) + s * Fraction(float(vi)) for gi, vi in zip(g, v)]
    return sorted(range(len(g)), key=lambda i: (w[i], i))


@pytest.mark.parametrize("ex", GOLD["count_n"])
def test_count_n_golden(orc, ex):
    g = np.array(ex["g"], np.int32)
    v = np.array(ex["v"], np.float32)
    idx = np.array(_line_sort(g, v, 1), np.int32)
    assert list(idx) == list(orc.sort(g + v.astype(np.float64)))
    O = orc.count_n(g, v, idx, ex["N"], 1, ex["t_dist"], ex["t_disp"])
    assert sorted(int(g[i]) for i in range(len(g)) if O[i] > 0) == ex["occluded_g"]


def _pair_exact(vq, vp, dk, s, t_dist, t_disp):
    # S7 (reading Q14): delta rounded once to fp32, the rest exact
    delta = np.float32(np.float32(vq) - np.float32(vp))
    if not Fraction(float(delta)) > Fraction(float(np.float32(t_disp))):
        return False
    return abs(dk + s * Fraction(float(delta))) < Fraction(float(np.float32(t_dist)))


def brute_n(orc, D, views, N, t_edge=1.0, t_dist=2.0, t_disp=0.5, max_scan=4096):
    H, W = D.shape
    lo, hi, _ = orc.stats(D)
    out = np.zeros((len(views), H, W), np.uint8)
    for vi, b in enumerate(views):
        s = max(abs(b[0]), abs(b[1]))
        h = orc.scan_length(lo, hi, s, max_scan) // 2
        if h == 0:
            continue
        cand = orc.candidates(D, b, t_edge)
        for cy, cx in zip(*np.nonzero(cand)):
            g, xs, ys, v = orc.scanline(D, b, (int(cx), int(cy)), h)
            order = _line_sort(g, v, s)
            n = len(order)
            for i, p in enumerate(order):
                for d in list(range(-(N // 2), 0)) + list(range(1, N // 2 + 1)):
                    if 0 <= i + d < n:
                        q = order[i + d]
                        if _pair_exact(v[q], v[p], int(g[q]) - int(g[p]), s, t_dist, t_disp):
                            out[vi, ys[p], xs[p]] = 1
                            break
    return out


@pytest.mark.parametrize("seed", range(6))
def test_detect_n_equals_python_brute(orc, seed):
    rng = scenes.SplitMix64(2101, seed)
    views = [(1, 0), (0, -1), (1, 1), (-2, 1), (2, 0)]
    for it in range(6):
        H, W = rng.randint(4, 12), rng.randint(4, 12)
        D = scenes.random_tiny_map(rng, H, W, ["int", "half", "noisy", "uniform"][it % 4])
        for N in (2, 4, 8):
            a = orc.detect(D, views, neighbors=N)
            b = brute_n(orc, D, views, N)
            assert (a == b).all(), (seed, it, N)


@pytest.mark.parametrize("seed", range(8))
def test_large_n_equals_infinity(orc, seed):
    rng = scenes.SplitMix64(2102, seed)
    views = scenes.all_small_baselines(2)
    for it in range(10):
        H, W = rng.randint(4, 20), rng.randint(4, 20)
        D = scenes.random_tiny_map(rng, H, W, ["int", "half", "noisy", "uniform"][it % 4])
        inf, info, _ = orc.detect(D, views, return_info=True)
        hmax = int(info[:, 2].max())
        Nbig = 2 * (2 * hmax + 1)
        assert (orc.detect(D, views, neighbors=Nbig) == inf).all()


@pytest.mark.parametrize("seed", range(4))
def test_monotone_in_n(orc, seed):
    rng = scenes.SplitMix64(2103, seed)
    views = [(1, 0), (-1, 0), (0, 1), (1, -1), (2, 1)]
    for it in range(8):
        H, W = rng.randint(6, 18), rng.randint(6, 18)
        D = scenes.random_tiny_map(rng, H, W, ["int", "half", "noisy", "uniform"][it % 4])
        prev = None
        for N in (2, 4, 6, 8, 16, 0):
            m = orc.detect(D, views, neighbors=N)
            if prev is not None:
                assert (m >= prev).all(), (seed, it, N)
            prev = m


def test_n_small_can_miss(orc):
    # the N = 2 golden case shows truncation matters; here a whole map: a
    # disparity step seen by a horizontal view at N = 2 marks a subset of N = inf
    D = np.zeros((4, 16), np.float32)
    D[:, 8:] = 3.0
    a = orc.detect(D, [(1, 0)], neighbors=2)
    b = orc.detect(D, [(1, 0)])
    assert (a <= b).all() and b.sum() > 0


def test_detect_n_validation(orc):
    D = np.zeros((4, 4), np.float32)
    for N in (1, 3, -2, 7):
        with pytest.raises(ValueError):
            orc.detect(D, [(1, 0)], neighbors=N)
    assert (orc.detect(D, [(1, 0)], neighbors=0) == orc.detect(D, [(1, 0)])).all()
