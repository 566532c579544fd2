"""Oracle pinned to the worked examples printed in SPEC.md (tests/golden/).

PAPER.md prints no numeric example (Fig. 2's images are absent); SPEC.md's
hand-computed examples restate PAPER.md §3's equations on tiny inputs.  Each
fixture in tests/golden/spec_examples.json carries its SPEC.md line.
"""
import json
import os

import numpy as np
import pytest

from paper_2408_14050_b200 import scenes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["stats"])
def test_stats(orc, ex):
    lo, hi, bad = orc.stats(np.array(ex["D"], np.float32))
    assert (lo, hi, bad) == (ex["min"], ex["max"], 0), ex["cite"]


@pytest.mark.parametrize("ex", GOLD["scan_length"])
def test_scan_length(orc, ex):
    assert orc.scan_length(ex["dmin"], ex["dmax"], 1, ex["cap"]) == ex["L"], ex["cite"]


def test_edges_row(orc):
    ex = GOLD["edges"][0]
    D = np.array([ex["row"], ex["row"]], np.float32)
    Ex, Ey, E = orc.edges(D)
    assert Ex[0, ex["index"]] == ex["Ex"] and E[0, ex["index"]] == ex["E"], ex["cite"]


def test_edges_constant_and_ramp(orc):
    # SPEC.md:115 constant -> all zero; SPEC.md:116 ramp D=x -> Ex=1 except last column
    Ex, Ey, E = orc.edges(np.full((5, 7), 5.0, np.float32))
    assert not Ex.any() and not Ey.any() and not E.any()
    D = np.tile(np.arange(7, dtype=np.float32), (5, 1))
    Ex, Ey, E = orc.edges(D)
    assert (Ex[:, :-1] == 1).all() and (Ex[:, -1] == 0).all() and not Ey.any()
    assert (E[:, :-1] == 1).all()


def test_scanline_axis(orc):
    ex = GOLD["scanline"][0]
    D = np.zeros((40, 100), np.float32)
    g, xs, ys, v = orc.scanline(D, tuple(ex["b"]), tuple(ex["c"]), ex["L"] // 2)
    assert list(xs) == ex["xs"] and (ys == ex["ys_const"]).all(), ex["cite"]
    assert list(g) == list(range(-8, 9))


def test_scanline_diagonal_step(orc):
    ex = GOLD["scanline"][1]
    D = np.zeros((30, 30), np.float32)
    g, xs, ys, v = orc.scanline(D, tuple(ex["b"]), tuple(ex["c"]), 2)
    i = list(g).index(ex["g"])
    assert [xs[i], ys[i]] == ex["xy"], ex["cite"]
    # digital line (reading Q8): g = 2 is (12, 12), no repeated pixel
    i2 = list(g).index(2)
    assert [xs[i2], ys[i2]] == [12, 12]


@pytest.mark.parametrize("ex", GOLD["sort"])
def test_sort(orc, ex):
    assert list(orc.sort(ex["w"])) == ex["idx"], ex["cite"]


@pytest.mark.parametrize("ex", GOLD["count"])
def test_count(orc, ex):
    idx = orc.sort(ex["w"])
    O = orc.count(ex["g"], ex["v"], ex["w"], idx, 1, ex["t_dist"], ex["t_disp"])
    occluded = [g for g, o in zip(ex["g"], O) if o > 0]
    assert occluded == ex["occluded_g"], ex["cite"]


def test_step_scene_detect(orc):
    ex = GOLD["step_detect"][0]
    D = scenes.step_scene(ex["H"], ex["W"], ex["bg"], ex["fg"], ex["col"], axis=0, fg_first=True)
    cand = orc.candidates(D, tuple(ex["b_occluding"]))
    ys, xs = np.nonzero(cand)
    assert (xs == ex["cand_col"]).all() and len(ys) == ex["H"], ex["cite"]
    assert not orc.candidates(D, tuple(ex["b_empty"])).any()
    m = orc.detect(D, [tuple(ex["b_occluding"]), tuple(ex["b_empty"])])
    lo, hi = ex["band"]
    expect = np.zeros((ex["H"], ex["W"]), np.uint8)
    expect[:, lo:hi + 1] = 1
    assert (m[0] == expect).all(), ex["cite"]
    assert not m[1].any()   # exactly one of two opposite masks is non-empty


def test_constant_map_all_directions(orc):
    # SPEC.md:218, 479 (acceptance 3): zero masks, zero candidates, L = 0
    m, info, rc = orc.detect(np.full((20, 30), 3.0, np.float32), scenes.VIEWS_3X3, return_info=True)
    assert rc == 0 and not m.any()
    assert (info[:, 0] == 0).all() and (info[:, 1] == 0).all()


def test_single_direction_consistency(orc):
    # detect_array with one direction equals detect
    D = scenes.make_scene(2)
    m8 = orc.detect(D, scenes.VIEWS_3X3)
    for i, b in enumerate(scenes.VIEWS_3X3[:3]):
        assert (orc.detect(D, [b])[0] == m8[i]).all()
