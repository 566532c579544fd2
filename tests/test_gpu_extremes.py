"""GPU parity at fp32 extremes: disparities near +-FLT_MAX make the forward
differences overflow to +-inf (Eq. 1), the frame range R overflow (Eq. 3: h
capped by max_scan), and the Eq. 2 dot products of the grid families produce
inf - inf = NaN (no candidate).  The candidate codes of K0 (generic and the
3x3 fast path), the line sweep's fallbacks and the per-pixel kernel must
agree with the oracle bit for bit."""
import numpy as np
import pytest

import oracle
from paper_2408_14050_b200 import scenes

from test_gpu_parity import assert_same, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2408_14050_b200 import build
    build.build()
    return torch


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("views", [scenes.VIEWS_3X3, [(1, 0), (2, 1), (0, -1)]])
def test_near_flt_max(torch_cuda, seed, views):
    rng = scenes.SplitMix64(7101, seed)
    H, W = 64, 160          # > 2^16 pixel-views: the K0 + line-sweep path, not the tiny-call kernel
    u = rng.uniform(H * W).reshape(H, W)
    D = np.where(u < 0.3, -3.0e38, np.where(u < 0.6, 3.0e38, 1.0e37 * (u - 0.8))).astype(np.float32)
    for max_scan in (9, 64, 150):     # h = 4 (per-pixel fallback), 32 and 75 (sweep)
        g, st = run_gpu(torch_cuda, D, views, max_scan=max_scan)
        assert st == [0]
        assert_same(g[0], oracle.detect(D, views, max_scan=max_scan), f"seed {seed} cap {max_scan}")
