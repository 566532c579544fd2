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
    H, W = 96, 256          # > 2^16 pixel-views for both view sets: K0 + line sweep / k_tile, not the tiny-call kernel
    assert H * W * len(views) > 1 << 16
    u = rng.uniform(H * W).reshape(H, W)
    D = np.where(u < 0.3, -3.0e38, np.where(u < 0.6, 3.0e38, 1.0e37 * (u - 0.8))).astype(np.float32)
    for max_scan in (9, 64, 150):     # h = 4 (per-pixel fallback), 32 and 75 (sweep)
        g, st = run_gpu(torch_cuda, D, views, max_scan=max_scan)
        assert st == [0]
        assert_same(g[0], oracle.detect(D, views, max_scan=max_scan), f"seed {seed} cap {max_scan}")


def test_knight_dot_overflow(torch_cuda):
    """the Eq. 2 dot of a knight family, 2 E_x + E_y with
    E_x = 2e38 and E_y = -inf, is -inf exactly (binary64);
    an fp32 product 2 * 2e38 overflows to +inf and the sum would be NaN.
    Pixel (20, 2) is then the only (-2,-1) candidate on its line."""
    H, W = 64, 160
    D = np.zeros((H, W), np.float32)
    D[:, 21:] = 3e38
    D[3:, :21] = -3e38
    D[2, 20] = 1e38
    D[0, 17] = D[0, 18] = D[1, 17] = 1.0
    views = scenes.VIEWS_5X5
    assert H * W * len(views) > 1 << 16          # K0 + k_line / k_tile, not the per-pixel kernel
    o = oracle.detect(D, views, max_scan=150)
    k = views.index((-2, -1))
    assert o[k][1, 18] == 1 and o[k][1, 19] == 1   # the marks only that candidate produces
    for path in ("auto", "tiled"):
        g, st = run_gpu(torch_cuda, D, views, max_scan=150, path=path)
        assert st == [0]
        for i, b in enumerate(views):
            assert_same(g[0, i], o[i], f"{path} view {b}")
