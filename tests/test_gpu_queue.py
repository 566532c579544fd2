"""GPU parity when the far-partner queue (line sweep -> k_hard, Eq. 5 far
pairs) overflows its capacity.

OCC_GQ_CAP (read at occ_create) shrinks the queue to a few entries, so that
most warps' reservations land beyond the capacity or straddle it: the entries
below the capacity must all be written by this call (k_hard reads every slot
below min(count, cap)), the rest resolved in the sweep warp.  Two consecutive
calls on one context catch stale slots of an earlier call."""
import os

import numpy as np
import pytest

import oracle
from paper_2408_14050_b200 import scenes

from test_gpu_parity import assert_same

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2408_14050_b200 import build
    build.build()
    return torch


@pytest.mark.parametrize("cap", [1, 37, 1000, 5000])
def test_forced_queue_overflow(torch_cuda, cap, monkeypatch):
    torch = torch_cuda
    from paper_2408_14050_b200.occ import Detector
    monkeypatch.setenv("OCC_GQ_CAP", str(cap))
    a = scenes.make_scene(3)[200:520, 600:1100].copy()       # noisy C3 crop: many far survivors
    b = scenes.make_scene(3, frame=1)[100:420, 900:1400].copy()
    views = scenes.VIEWS_3X3
    H, W = a.shape
    det = Detector(H, W, views, max_batch=2)
    monkeypatch.delenv("OCC_GQ_CAP")
    oa = oracle.detect(a, views)
    ob = oracle.detect(b, views)
    for D, o in ((np.stack([a, b]), (oa, ob)), (np.stack([b, a]), (ob, oa))):   # two calls, one ctx
        m = det.detect(torch.from_numpy(D).cuda())
        torch.cuda.synchronize()
        assert det.status() == [0, 0]
        g = m.cpu().numpy()
        for f in range(2):
            for i, v in enumerate(views):
                assert_same(g[f, i], o[f][i], f"cap {cap} frame {f} view {v}")
    det.close()
