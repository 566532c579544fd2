"""Oracle pinned to closed forms and exact arithmetic (not to itself).

* S7 pair predicate vs exact rational arithmetic (fractions.Fraction).
* S4 exact sign test vs the literal two-argument-arctangent form of Eq. 2.
* S3 literal fp32 magnitude (numpy float32 ops) vs the oracle's E.
* Eq. 3-6 step and rectangle closed forms (derived by hand
  from PAPER.md Eqs. 3-6; BASELINE.json north_star: "an occluded band of
  width (d_fg - d_bg)*|baseline| on the background side").
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from paper_2408_14050_b200 import scenes


def exact_pair(vq, vp, dk, s, t_dist, t_disp):
    delta = np.float32(np.float32(vq) - np.float32(vp))   # one fp32 rounding (Q14)
    if not (delta > np.float32(t_disp)):
        return 0
    if not np.isfinite(delta):
        return 0
    w = Fraction(dk) + s * Fraction(float(delta))
    return int(abs(w) < Fraction(float(np.float32(t_dist))))


def test_pair_predicate_exact(orc):
    rng = scenes.SplitMix64(7, 7)
    n = 0
    for _ in range(4000):
        s = rng.randint(1, 8)
        dk = rng.randint(-40, 40)
        t_dist = float(np.float32([0.5, 1.0, 2.0, 1.7, 3.25, 0.3][rng.randint(0, 5)]))
        t_disp = [0.0, 0.5, 0.25, 1.0][rng.randint(0, 3)]
        vp = np.float32(rng.uniform_range(-10, 60))
        # hit the interval boundaries: delta near (dk +- t)/s
        target = (-dk + (t_dist if rng.randint(0, 1) else -t_dist)) / s
        vq = np.float32(vp + target + (rng.uniform_range(-1, 1) * 10 ** -rng.randint(0, 7)))
        assert orc.pair(float(vq), float(vp), dk, s, t_dist, t_disp) == exact_pair(vq, vp, dk, s, t_dist, t_disp)
        n += exact_pair(vq, vp, dk, s, t_dist, t_disp)
    assert n > 200   # the sweep exercised both outcomes


def test_pair_predicate_boundaries(orc):
    # |dk + s delta| < t is strict; delta > t_disp is strict (reading Q3/Q13)
    assert orc.pair(3.0, 1.0, 0, 1, 2.0, 0.5) == 0      # |0 + 2| = 2 not < 2
    assert orc.pair(3.0, 1.0, -1, 1, 2.0, 0.5) == 1
    assert orc.pair(1.5, 1.0, 0, 1, 2.0, 0.5) == 0      # delta = 0.5 not > 0.5
    assert orc.pair(1.0, 3.0, -2, 1, 2.0, 0.5) == 0     # smaller neighbour never occludes
    nxt = float(np.nextafter(np.float32(3.0), np.float32(0)))
    assert orc.pair(nxt, 1.0, 0, 1, 2.0, 0.5) == 1      # just below the bound


def test_candidate_sign_matches_angle_form(orc):
    # Eq. 2 with Theta = atan2(Ey, Ex), circular |Theta - phi| < pi/2, away from
    # the pi/2 boundary where binary64 atan2 may round either way.
    rng = scenes.SplitMix64(11)
    for _ in range(3000):
        ex = np.float32(rng.uniform_range(-5, 5))
        ey = np.float32(rng.uniform_range(-5, 5))
        bx, by = rng.randint(-8, 8), rng.randint(-8, 8)
        if bx == 0 and by == 0:
            continue
        dot = float(ex) * bx + float(ey) * by
        if abs(dot) < 1e-6 * math.hypot(bx, by) * math.hypot(float(ex), float(ey)) + 1e-30:
            continue
        D = np.zeros((2, 2), np.float32)
        D[0, 1] = ex
        D[1, 0] = ey
        c = orc.candidates(D, (bx, by), t_edge=1e-30)[0, 0]
        assert c == orc.angle_predicate(float(ex), float(ey), (bx, by))
        assert c == (dot > 0)


def test_magnitude_literal_fp32(orc):
    rng = scenes.SplitMix64(12)
    D = (rng.uniform(64 * 64) * 10).astype(np.float32).reshape(64, 64)
    Ex, Ey, E = orc.edges(D)
    ex = np.zeros_like(D); ex[:, :-1] = D[:, 1:] - D[:, :-1]
    ey = np.zeros_like(D); ey[:-1, :] = D[1:, :] - D[:-1, :]
    e = np.sqrt((ex * ex).astype(np.float32) + (ey * ey).astype(np.float32)).astype(np.float32)
    assert (Ex == ex).all() and (Ey == ey).all() and (E == e).all()


def test_scan_length_scaling_and_rounding(orc):
    # Eq. 3: L = ceil(2 s (max - min)), fl32 range, capped
    assert orc.scan_length(1.0, 48.0, 2, 4096) == 188
    assert orc.scan_length(1.0, 48.0, 1, 4096) == 94
    assert orc.scan_length(0.0, 0.3, 1, 4096) == 1        # ceil(0.6) = 1 -> h = 0
    assert orc.scan_length(-3.0e38, 3.0e38, 1, 4096) == 4096   # fl32 overflow -> cap
    R = np.float32(np.float32(7.1) - np.float32(2.05))
    assert orc.scan_length(2.05, 7.1, 3, 4096) == math.ceil(2 * 3 * Fraction(float(R)))


def expected_step_band(W, e, delta, s, fg_high_side, sign, t_dist):
    """App. A.4 closed form along the major axis for a step at pixel boundary
    e-1 | e.  fg_high_side: fg occupies positions >= e.  sign: sign of the
    baseline's major component.  Returns (lo, hi) inclusive or None."""
    h = s * delta
    if sign > 0 and fg_high_side:          # occluders at larger position
        width = s * delta + (1 if t_dist > 1 else 0)
        return max(0, e - width), e - 1
    if sign < 0 and not fg_high_side:      # occluders at smaller position
        width = s * delta + (1 if (t_dist > 1 and h >= s * delta + 1) else 0)
        return e, min(W - 1, e + width - 1)
    return None


@pytest.mark.parametrize("s", [1, 2])
@pytest.mark.parametrize("sign", [1, -1])
@pytest.mark.parametrize("fg_high", [True, False])
@pytest.mark.parametrize("t_dist", [0.5, 1.0, 2.0])
@pytest.mark.parametrize("axis", [0, 1])
def test_step_closed_form(orc, s, sign, fg_high, t_dist, axis):
    H, W, e, bg, fg = 24, 64, 30, 1.0, 6.0
    delta = int(fg - bg)
    if axis == 0:
        D = scenes.step_scene(H, W, bg, fg, e, axis=0, fg_first=not fg_high)
        b = (sign * s, 0)
    else:
        D = scenes.step_scene(W, H, bg, fg, e, axis=1, fg_first=not fg_high)
        b = (0, sign * s)
    m = orc.detect(D, [b], t_dist=t_dist)[0]
    band = expected_step_band(W, e, delta, s, fg_high, sign, t_dist)
    expect = np.zeros((H, W), np.uint8)
    if band is not None:
        expect[:, band[0]:band[1] + 1] = 1
    if axis == 1:
        expect = expect.T
    assert (m == expect).all()


def test_config1_exact_mask(orc):
    # C1 (BASELINE.json configs[0]): 20x16 rect at 8 on bg 2, b = (+1, 0):
    # band columns [x0-7, x0-1] x rows [y0, y0+15] = 112 px at t_dist = 2,
    # [x0-6, x0-1] = 96 px at t_dist <= 1 (the z-buffer band, Delta*|b| = 6).
    D = scenes.make_scene(1)
    x0, y0 = scenes.c1_rect_origin()
    assert D[y0, x0] == 8 and D[y0 - 1 if y0 else y0 + 16, x0] == 2
    for t_dist, width in ((2.0, 7), (1.0, 6), (0.75, 6)):
        m, info, rc = orc.detect(D, [(1, 0)], t_dist=t_dist, return_info=True)
        expect = np.zeros_like(m[0])
        expect[y0:y0 + 16, x0 - width:x0] = 1
        assert (m[0] == expect).all()
        assert tuple(info[0]) == (16, 12, 6, 16 * width)


def test_diagonal_step_interior_width(orc):
    # App. A.4: oblique baselines give the same width along the major axis in
    # the interior (rows whose scan lines stay inside the image).
    H, W, e = 60, 60, 30
    D = scenes.step_scene(H, W, 1.0, 5.0, e, axis=0, fg_first=False)
    m = orc.detect(D, [(1, 1), (1, -1), (2, 1)])
    for i, (b, s) in enumerate((((1, 1), 1), ((1, -1), 1), ((2, 1), 2))):
        width = s * 4 + 1
        rows = range(12, H - 12)
        for y in rows:
            xs = np.nonzero(m[i][y])[0]
            assert list(xs) == list(range(e - width, e)), (b, y, xs)


def test_nonfinite_and_validation(orc):
    D = np.ones((8, 8), np.float32)
    D[3, 3] = np.nan
    m, info, rc = orc.detect(D, [(1, 0)], return_info=True)
    assert rc == orc.ERR_NONFINITE and not m.any()
    D[3, 3] = np.inf
    assert orc.detect(D, [(1, 0)], return_info=True)[2] == orc.ERR_NONFINITE
    assert orc.validate(1, 8, [(1, 0)]) == orc.ERR_INVALID_ARG
    assert orc.validate(8, 8, []) == orc.ERR_INVALID_ARG
    assert orc.validate(8, 8, [(0, 0)]) == orc.ERR_INVALID_ARG
    assert orc.validate(8, 8, [(9, 0)]) == orc.ERR_UNSUPPORTED
    assert orc.validate(8, 8, [(1, 0)], t_edge=0.0) == orc.ERR_INVALID_ARG
    assert orc.validate(8, 8, [(1, 0)], t_dist=0.0) == orc.ERR_INVALID_ARG
    assert orc.validate(8, 8, [(1, 0)], t_disp=-1.0) == orc.ERR_INVALID_ARG
    assert orc.validate(8, 8, [(1, 0)], max_scan=0) == orc.ERR_INVALID_ARG
    assert orc.validate(8, 8, [(1, 0)]) == orc.OK


def test_h_zero_gives_empty(orc):
    # Eq. 3 with range 0.3: L = 1, h = 0 -> every scan line is the candidate alone
    D = np.zeros((6, 6), np.float32)
    D[:, 3:] = 0.3
    m, info, rc = orc.detect(D, [(1, 0)], t_edge=0.1, t_disp=0.1, return_info=True)
    assert info[0, 0] > 0 and info[0, 2] == 0 and not m.any()
