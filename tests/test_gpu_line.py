"""GPU parity of the line-sweep kernel k_line (+ k_hard) against the oracle.

k_line serves the +-b view pairs of the row / column / diagonal /
anti-diagonal families whenever the frame's scan half-length satisfies
17 <= h <= 96; other frames take its in-kernel per-pixel
fallback.  These cases drive the sweep itself: moderate sizes with disparity
ranges that put h in that window, ragged widths (no 16-byte row alignment,
partial line blocks, W % 4 != 0), single-view groups (+b or -b alone), s = 2
pairs, thin occluders (true misses for the k_hard queue), and agreement with
the tiled kernel.  Bit-exact (uint8 masks).
"""
import numpy as np
import pytest

import oracle
from paper_2408_14050_b200 import scenes

from test_gpu_parity import assert_same, run_gpu

pytestmark = pytest.mark.gpu

LINE_VIEWS = [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1), (1, -1), (-1, 1),
              (2, 0), (-2, 0), (0, 2), (2, 2), (-2, 2)]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2408_14050_b200 import build
    build.build()
    return torch


def layered(rng, H, W, n, lo, hi, noise):
    """Painter's-order rectangles over a slanted plane (values in [lo, hi])."""
    y = np.arange(H, dtype=np.float64)[:, None]
    img = np.broadcast_to(lo + 2.0 * y / max(1, H - 1), (H, W)).copy()
    shapes = []
    for i in range(n):
        u = rng.uniform(5)
        cx, cy = u[0] * (W - 1), u[1] * (H - 1)
        ax, ay = 1 + u[2] * W / 5, 1 + u[3] * H / 5
        shapes.append((lo + (hi - lo) * u[4], i, cx, cy, ax, ay))
    shapes.sort()
    for d, _, cx, cy, ax, ay in shapes:
        x0, x1 = max(0, int(cx - ax)), min(W, int(cx + ax) + 1)
        y0, y1 = max(0, int(cy - ay)), min(H, int(cy + ay) + 1)
        img[y0:y1, x0:x1] = d
    if noise:
        img = img + noise * rng.normal(H * W).reshape(H, W)
    return img.astype(np.float32)


SIZES = [(70, 90), (33, 200), (130, 50), (64, 64), (97, 131), (40, 257)]


@pytest.mark.parametrize("H,W", SIZES)
@pytest.mark.parametrize("noise", [0.0, 0.25])
def test_line_sweep_random_layers(torch_cuda, H, W, noise):
    rng = scenes.SplitMix64(1201, H, W, int(noise * 100))
    # disparities in [1, 45]: h in [17, 96] for s = 1 and s = 2
    D = np.stack([layered(rng, H, W, 12, 1.0, 45.0, noise) for _ in range(3)])
    g, st = run_gpu(torch_cuda, D, LINE_VIEWS)
    assert st == [0, 0, 0]
    for f in range(len(D)):
        assert_same(g[f], oracle.detect(D[f], LINE_VIEWS), f"{H}x{W} noise {noise} frame {f}")


@pytest.mark.parametrize("views", [[(1, 0)], [(-1, 0)], [(0, -1), (1, 1)], [(-1, 1), (2, 0)],
                                   [(1, 0), (2, 0)], [(0, 1), (0, -2)]])
def test_line_sweep_single_view_groups(torch_cuda, views):
    rng = scenes.SplitMix64(1202, len(views), views[0][0] + 3 * views[0][1])
    D = np.stack([layered(rng, 80, 120, 10, 1.0, 40.0, 0.25) for _ in range(2)])
    g, _ = run_gpu(torch_cuda, D, views)
    for f in range(len(D)):
        assert_same(g[f], oracle.detect(D[f], views), f"{views} frame {f}")


def test_line_sweep_thin_occluders(torch_cuda):
    # 1-3 pixel wide high-disparity bars over a noisy background: far filter
    # survivors without partners (the k_hard queue) and bands cut short
    rng = scenes.SplitMix64(1203)
    H, W = 96, 160
    D = 2.0 + 0.25 * rng.normal(H * W).reshape(H, W)
    for i in range(14):
        u = rng.uniform(4)
        x, y = int(u[0] * (W - 4)), int(u[1] * (H - 30))
        wdt = 1 + int(u[2] * 3)
        D[y:y + 25, x:x + wdt] = 20.0 + 20.0 * u[3]
        D[y + int(u[3] * 20), max(0, x - 20):x + 20] = 30.0 + 10.0 * u[2]
    D = D.astype(np.float32)
    g, _ = run_gpu(torch_cuda, D, LINE_VIEWS)
    assert_same(g[0], oracle.detect(D, LINE_VIEWS), "thin occluders")


def test_line_vs_tiled_paths(torch_cuda):
    D = np.ascontiguousarray(scenes.make_batch(3, 2)[:, 200:520, 300:900])
    views = scenes.VIEWS_3X3
    a, _ = run_gpu(torch_cuda, D, views, path="auto")
    b, _ = run_gpu(torch_cuda, D, views, path="tiled")
    assert (a == b).all()
    assert_same(a[0], oracle.detect(D[0], views), "C3 crop")


def test_host_pipeline_multiple_chunks(torch_cuda, monkeypatch):
    # 48 MiB chunks of 1080p frames hold 4 frames, so 7 frames = two chunks (4 + 3)
    from paper_2408_14050_b200.occ import Detector
    monkeypatch.setenv("OCC_CHUNK_MIB", "48")
    D = scenes.make_batch(5, 7)
    views = scenes.config_views(5)
    det = Detector(1080, 1920, views, max_batch=7)
    mh = det.detect_host(D)
    assert det.status() == [0] * 7
    det.close()
    dev, _ = run_gpu(torch_cuda, D, views)
    assert (mh == dev).all()
    for i, b in enumerate(views[:3]):
        assert_same(mh[6, i], oracle.detect(D[6], [b])[0], f"frame 6 view {b}")
