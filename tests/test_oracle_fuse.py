"""Pins of the oracle's median fusion (PAPER.md:238,
SPEC.md:51-58): SPEC's printed examples, the textbook definition written out
on tiny stacks, order invariance, identity on copies, the even-count fp32
recipe, and non-finite propagation."""
import itertools
import json
import os

import numpy as np

import oracle
from paper_2408_14050_b200 import scenes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_spec_examples():
    for ex in GOLD["fuse_median"]:
        if "values" in ex:
            st = np.array(ex["values"], np.float32).reshape(-1, 1)
            assert oracle.fuse_median(st)[0] == ex["median"], ex["cite"]
        else:
            st = np.array(ex["stack"], np.float32)
            assert (oracle.fuse_median(st) == np.array(ex["out"], np.float32)).all(), ex["cite"]


def textbook(vals):
    """Median by definition: sort, middle element, or mean of the middle pair."""
    v = sorted(float(x) for x in vals)
    k = len(v)
    if k % 2:
        return np.float32(v[k // 2])
    return np.float32(np.float32(np.float32(v[k // 2 - 1]) + np.float32(v[k // 2])) * np.float32(0.5))


def test_textbook_definition_random():
    rng = scenes.SplitMix64(77)
    for K in list(range(1, 12)) + [16, 17]:
        st = ((rng.uniform(K * 50) - 0.5) * 200).astype(np.float32).reshape(K, 50)
        got = oracle.fuse_median(st)
        for p in range(50):
            assert got[p] == textbook(st[:, p]), (K, p)


def test_ties_and_integers():
    rng = scenes.SplitMix64(78)
    for K in (2, 4, 6, 8):
        st = np.floor(rng.uniform(K * 40) * 4).astype(np.float32).reshape(K, 40)
        got = oracle.fuse_median(st)
        ref = np.array([textbook(st[:, p]) for p in range(40)], np.float32)
        assert (got == ref).all()


def test_order_invariance():
    rng = scenes.SplitMix64(79)
    st = rng.normal(6 * 30).astype(np.float32).reshape(6, 30)
    base = oracle.fuse_median(st)
    for perm in itertools.permutations(range(6)):
        assert (oracle.fuse_median(st[list(perm)]) == base).all()


def test_copies_identity():
    D = scenes.make_scene(2)[:40, :60]
    for K in (1, 2, 3, 8):
        assert (oracle.fuse_median(np.stack([D] * K)) == D).all()


def test_even_count_rounding():
    # fl32(a + b) then exact halving: a + b = 1 + 2^-24 rounds to 1 before halving
    a, b = np.float32(0.5), np.float32(0.5 + 2.0 ** -24)
    st = np.array([[a], [b]], np.float32)
    assert oracle.fuse_median(st)[0] == np.float32(np.float32(a + b) * np.float32(0.5))
    # large values: the mean stays finite (no overflow of a + b for disparities)
    st = np.array([[1e30], [3e30]], np.float32)
    assert oracle.fuse_median(st)[0] == np.float32(2e30)


def test_nonfinite_propagates():
    st = np.ones((5, 4), np.float32)
    st[2, 1] = np.nan
    st[4, 3] = np.inf
    out = oracle.fuse_median(st)
    assert out[0] == 1 and out[2] == 1 and np.isnan(out[1]) and np.isnan(out[3])
