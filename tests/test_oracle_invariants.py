"""Exact invariants of the defined detector.

* transpose equivariance: M(D^T, (by, bx)) = M(D, (bx, by))^T  (digital lines
  of S6 are transpose-symmetric; Eq. 1's forward difference is too)
* half-plane partition of candidates
* threshold monotonicity: smaller t_e / t_disp or larger t_dist / cap
  give supersets (each enlarges the sets in Eqs. 2, 5 or the windows of Eq. 4)
* integer offset invariance on integer maps (Eq. 1-6 use differences only)
* empty on planar fronto maps (constant D) and determinism
"""
import numpy as np
import pytest

from paper_2408_14050_b200 import scenes

MODES = ["int", "half", "noisy", "uniform"]


@pytest.mark.parametrize("mode", MODES)
def test_transpose_equivariance(orc, mode):
    rng = scenes.SplitMix64(301, MODES.index(mode))
    views = scenes.all_small_baselines(2) + [(3, 1), (-1, 4)]
    for _ in range(40):
        D = scenes.random_tiny_map(rng, rng.randint(4, 20), rng.randint(4, 20), mode)
        a = orc.detect(D, views)
        bt = orc.detect(np.ascontiguousarray(D.T), [(by, bx) for bx, by in views])
        assert (a == bt.transpose(0, 2, 1)).all()


def test_transpose_equivariance_c2(orc):
    D = scenes.make_scene(2)
    a = orc.detect(D, scenes.VIEWS_3X3)
    bt = orc.detect(np.ascontiguousarray(D.T), [(by, bx) for bx, by in scenes.VIEWS_3X3])
    assert (a == bt.transpose(0, 2, 1)).all()


def test_half_plane_partition(orc):
    rng = scenes.SplitMix64(302)
    D = scenes.random_tiny_map(rng, 30, 30, "noisy")
    _, _, E = orc.edges(D)
    Ex, Ey, _ = orc.edges(D)
    for b in scenes.all_small_baselines(2):
        cp = orc.candidates(D, b)
        cm = orc.candidates(D, (-b[0], -b[1]))
        assert not (cp & cm).any()
        perp = (b[0] * Ex.astype(np.float64) + b[1] * Ey.astype(np.float64)) == 0
        assert ((cp | cm).astype(bool) == ((E > 1.0) & ~perp)).all()


@pytest.mark.parametrize("knob", ["t_edge", "t_disp", "t_dist", "max_scan"])
def test_threshold_monotonicity(orc, knob):
    rng = scenes.SplitMix64(303, ["t_edge", "t_disp", "t_dist", "max_scan"].index(knob))
    views = scenes.all_small_baselines(2)
    pairs = {"t_edge": (2.0, 0.5), "t_disp": (1.0, 0.25), "t_dist": (1.0, 3.0), "max_scan": (6, 4096)}
    tight, loose = pairs[knob]
    grew = 0
    for it in range(30):
        D = scenes.random_tiny_map(rng, 16, 16, MODES[it % 4])
        a = orc.detect(D, views, **{knob: tight})
        b = orc.detect(D, views, **{knob: loose})
        assert (b >= a).all()
        grew += int((b > a).sum())
    assert grew > 0


def test_integer_offset_invariance(orc):
    rng = scenes.SplitMix64(304)
    for _ in range(30):
        D = scenes.random_tiny_map(rng, 16, 16, "int")
        off = float(rng.randint(-20, 20))
        a = orc.detect(D, scenes.all_small_baselines(2))
        b = orc.detect((D + off).astype(np.float32), scenes.all_small_baselines(2))
        assert (a == b).all()


def test_constant_and_determinism(orc):
    for v in (0.0, 7.5, -3.0):
        assert not orc.detect(np.full((9, 13), v, np.float32), scenes.all_small_baselines(2)).any()
    D = scenes.make_scene(2)
    assert (orc.detect(D, scenes.VIEWS_3X3) == orc.detect(D, scenes.VIEWS_3X3)).all()


def test_digital_line_partition(orc):
    # S6: every pixel lies on exactly one line per family and consecutive
    # samples differ by one in k; scan lines from any two pixels of a line
    # enumerate the same pixels.
    H, W = 13, 17
    D = np.arange(H * W, dtype=np.float32).reshape(H, W)
    for b in scenes.all_small_baselines(3):
        seen = np.zeros((H, W), np.int32)
        lines = {}
        for y in range(H):
            for x in range(W):
                g, xs, ys, v = orc.scanline(D, b, (x, y), H + W)
                key = tuple(sorted(zip(xs.tolist(), ys.tolist())))
                lines.setdefault(key, 0)
                assert (np.diff(g) == 1).all()
                assert (v == D[ys, xs]).all()
        for key in lines:
            for (x, y) in key:
                seen[y, x] += 1
        assert (seen == 1).all(), b
