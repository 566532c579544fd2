"""GPU parity of the finite-N detector (occ_set_neighbors, k_nwin; SURVEY
§8(f) NEXT #1) against the oracle's orc_detect_n, bit-exact.

Covered: N in {2, 4, 6, 8, 16} on random layered maps and random tiny maps
(every small baseline, knight moves, s = 2, 3), the SPEC.md:155 default N = 8
on a whole C2 / C3 frame and a C5 frame in the bench's launch configuration,
both mask formats, windows longer than the shared-memory capacity (h > 159:
global-scratch launch), a small max_scan cap, non-finite frames, multi-chunk
host pipeline, and a large N that must equal the N = infinity path.
"""
import numpy as np
import pytest

import oracle
from paper_2408_14050_b200 import scenes

from test_gpu_line import layered
from test_gpu_parity import assert_same

pytestmark = pytest.mark.gpu

MODES = ["int", "half", "noisy", "uniform"]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2408_14050_b200 import build
    build.build()
    return torch


def run(torch, D, views, N, fmt="u8", host=False, **kw):
    from paper_2408_14050_b200.occ import Detector, unpack_masks
    D = np.ascontiguousarray(D, np.float32)
    if D.ndim == 2:
        D = D[None]
    B, H, W = D.shape
    det = Detector(H, W, views, max_batch=B, mask_format=fmt, neighbors=N, **kw)
    if host:
        m = det.detect_host(D)
    else:
        m = det.detect(torch.from_numpy(D).cuda())
        torch.cuda.synchronize()
        m = m.cpu().numpy()
    st = det.status()
    det.close()
    if fmt == "bits":
        m = unpack_masks(m, W)
    return m, st


@pytest.mark.parametrize("N", [2, 4, 8, 16])
@pytest.mark.parametrize("H,W", [(70, 90), (33, 200), (97, 131)])
def test_nwin_layered(torch_cuda, N, H, W):
    rng = scenes.SplitMix64(3101, H, W, N)
    views = [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1), (2, 1), (-1, 2), (2, 0)]
    D = np.stack([layered(rng, H, W, 12, 1.0, 30.0, 0.25 * f) for f in range(2)])
    g, st = run(torch_cuda, D, views, N)
    assert st == [0, 0]
    for f in range(2):
        assert_same(g[f], oracle.detect(D[f], views, neighbors=N), f"{H}x{W} N={N} frame {f}")


@pytest.mark.parametrize("chunk", range(4))
def test_nwin_tiny_maps(torch_cuda, chunk):
    rng = scenes.SplitMix64(3102, chunk)
    views = scenes.all_small_baselines(2) + [(3, 1), (-1, 3)]
    for it in range(12):
        H, W = rng.randint(3, 24), rng.randint(3, 24)
        D = scenes.random_tiny_map(rng, H, W, MODES[it % 4])
        N = [2, 4, 6, 8][it % 4]
        kw = {} if it % 3 else dict(t_dist=[1.0, 0.5, 3.5][it % 3], t_disp=[0.25, 1.0, 0.5][it % 3])
        g, _ = run(torch_cuda, D, views, N, **kw)
        assert_same(g[0], oracle.detect(D, views, neighbors=N, **kw), f"chunk {chunk} it {it} N={N}")


@pytest.mark.parametrize("cfg", [2, 3])
def test_nwin_default_n_full_frame(torch_cuda, cfg):
    D = scenes.make_scene(cfg)
    views = scenes.config_views(cfg)
    g, st = run(torch_cuda, D, views, 8)
    o = oracle.detect(D, views, neighbors=8)
    for i, b in enumerate(views):
        assert_same(g[0, i], o[i], f"C{cfg} N=8 view {b}")


def test_nwin_c5_bench_launch(torch_cuda):
    # the launch configuration bench.py --neighbors 8 times: one call over a
    # batch of C5 frames; sampled frames vs the oracle
    D = scenes.make_batch(5, 6)
    views = scenes.config_views(5)
    g, st = run(torch_cuda, D, views, 8, fmt="bits")
    assert st == [0] * 6
    for f in (0, 5):
        o = oracle.detect(D[f], views, neighbors=8)
        for i, b in enumerate(views):
            assert_same(g[f, i], o[i], f"C5 frame {f} view {b}")


def test_nwin_packed_equals_u8(torch_cuda):
    rng = scenes.SplitMix64(3103)
    D = np.stack([layered(rng, 61, 157, 10, 1.0, 25.0, 0.25) for _ in range(3)])
    views = scenes.VIEWS_3X3 + [(2, 1)]
    a, _ = run(torch_cuda, D, views, 8)
    b, _ = run(torch_cuda, D, views, 8, fmt="bits")
    assert (a == b).all()


def test_nwin_long_windows(torch_cuda):
    # disparities over [1, 90] with s = 2: h = 178 > 159, windows of up to
    # 357 entries take the global-scratch launch; s = 1 views stay in smem
    rng = scenes.SplitMix64(3104)
    D = layered(rng, 48, 420, 14, 1.0, 90.0, 0.25)
    views = [(1, 0), (2, 0), (-2, 0), (0, 2), (2, 2), (2, -1)]
    for N in (2, 8):
        g, _ = run(torch_cuda, D, views, N)
        assert_same(g[0], oracle.detect(D, views, neighbors=N), f"long windows N={N}")


def test_nwin_small_max_scan(torch_cuda):
    rng = scenes.SplitMix64(3105)
    D = layered(rng, 50, 70, 8, 1.0, 20.0, 0.25)
    for cap in (1, 2, 9):
        g, _ = run(torch_cuda, D, scenes.VIEWS_3X3, 4, max_scan=cap)
        assert_same(g[0], oracle.detect(D, scenes.VIEWS_3X3, neighbors=4, max_scan=cap), f"max_scan {cap}")


def test_nwin_nonfinite_and_flat(torch_cuda):
    rng = scenes.SplitMix64(3106)
    D = np.stack([layered(rng, 40, 60, 6, 1.0, 20.0, 0.0) for _ in range(3)])
    D[1, 5, 7] = np.nan
    D[2] = 3.0                              # flat: h = 0, no marks
    g, st = run(torch_cuda, D, scenes.VIEWS_3X3, 8)
    assert st[1] != 0 and st[0] == 0 and st[2] == 0
    assert g[1].sum() == 0 and g[2].sum() == 0
    assert_same(g[0], oracle.detect(D[0], scenes.VIEWS_3X3, neighbors=8), "frame 0")


def test_nwin_large_n_equals_infinity(torch_cuda):
    from test_gpu_parity import run_gpu
    rng = scenes.SplitMix64(3107)
    D = np.stack([layered(rng, 64, 96, 10, 1.0, 20.0, 0.25) for _ in range(2)])
    views = scenes.VIEWS_3X3
    g, _ = run(torch_cuda, D, views, 2 * (2 * 40 + 1))    # h <= 38 here
    inf, _ = run_gpu(torch_cuda, D, views)
    assert (g == inf).all()


def test_nwin_host_pipeline(torch_cuda, monkeypatch):
    monkeypatch.setenv("OCC_CHUNK_MIB", "48")
    D = scenes.make_batch(5, 5)
    views = scenes.config_views(5)
    h, st = run(torch_cuda, D, views, 8, host=True)
    d, _ = run(torch_cuda, D, views, 8)
    assert st == [0] * 5
    assert (h == d).all()


def test_nwin_argument_validation(torch_cuda):
    from paper_2408_14050_b200.occ import Detector, OccError
    det = Detector(16, 16, [(1, 0)])
    for N in (-2, 1, 3, 7, 65538):
        with pytest.raises(OccError):
            det.set_neighbors(N)
    det.set_neighbors(8)
    det.set_neighbors(0)
    det.close()
