"""GPU side of single-frame spatial sharding (NEXT #4): occ_frame_stats is
exact, and row bands extended by the 2h + 2 halo and detected with the
imposed whole-frame statistics (occ_set_frame_stats) reproduce the whole
frame bit for bit -- the ranks are emulated one after another on the one
GPU (the NCCL exchange itself is covered by the gloo tests)."""
import numpy as np
import pytest

import oracle
from paper_2408_14050_b200 import scenes, spatial

from test_spatial import VIEWS, frame

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2408_14050_b200 import build
    build.build()
    return torch


def test_frame_stats_exact(torch_cuda):
    from paper_2408_14050_b200.occ import Detector
    D = np.stack([frame(s) for s in range(3)])
    D[2, 4, 4] = np.inf
    det = Detector(D.shape[1], D.shape[2], VIEWS, max_batch=3)
    lo, hi, bad = det.frame_stats(torch_cuda.from_numpy(D).cuda())
    det.close()
    for f in range(3):
        olo, ohi, obad = oracle.stats(D[f])
        assert (lo[f], hi[f], bad[f]) == (np.float32(olo), np.float32(ohi), obad)


def emulate(torch, D, world, views, N=0, fmt="u8"):
    H = D.shape[0]
    stats_fn, detect_fn, h_fn, close = spatial.device_fns(views, neighbors=N, mask_format=fmt)
    los, his, bads = zip(*[stats_fn(torch.from_numpy(D[r0:r1].copy()).cuda()) for r0, r1 in spatial.bands(H, world)])
    dmin, dmax, nbad = min(los), max(his), sum(bads)
    halo = 0 if nbad else spatial.halo_rows(h_fn(dmin, dmax))
    parts = []
    for r0, r1 in spatial.bands(H, world):
        e0, e1 = spatial.extended(r0, r1, halo, H)
        m = detect_fn(torch.from_numpy(D[e0:e1].copy()).cuda(), dmin, dmax, nbad)
        parts.append(m[:, r0 - e0:r1 - e0].cpu().numpy())
    close()
    return np.concatenate(parts, axis=1)


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("N", [0, 8])
def test_bands_equal_whole_frame(torch_cuda, world, N):
    from test_gpu_parity import run_gpu
    D = frame(11)
    got = emulate(torch_cuda, D, world, VIEWS, N)
    if N == 0:
        whole, _ = run_gpu(torch_cuda, D, VIEWS)
        assert (got == whole[0]).all()
    assert (got == oracle.detect(D, VIEWS, neighbors=N)).all()


def test_bands_c3_crop_packed(torch_cuda):
    from paper_2408_14050_b200.occ import unpack_masks
    D = np.ascontiguousarray(scenes.make_scene(3)[:400, :640])
    got = emulate(torch_cuda, D, 3, scenes.VIEWS_3X3, fmt="bits")
    ref = oracle.detect(D, scenes.VIEWS_3X3)
    assert (unpack_masks(got, 640) == ref).all()


def test_bands_nonfinite(torch_cuda):
    D = frame(12)
    D[80, 3] = np.nan
    assert emulate(torch_cuda, D, 3, VIEWS).sum() == 0


def test_scan_half_lengths_match_oracle(torch_cuda):
    """occ_scan_half_lengths (Eq. 3) vs the oracle's scan length."""
    from paper_2408_14050_b200.occ import Detector
    views = scenes.VIEWS_5X5
    det = Detector(16, 16, views, max_scan=300)
    for lo, hi in [(1.0, 12.3), (0.0, 0.0), (-3.5, 64.9), (1.0, 3000.0), (-3e38, 3e38)]:
        got = det.scan_half_lengths(lo, hi)
        want = [oracle.scan_length(lo, hi, max(abs(bx), abs(by)), 300) // 2 for bx, by in views]
        assert got == want, (lo, hi)
    det.close()
