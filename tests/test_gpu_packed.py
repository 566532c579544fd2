"""GPU parity of the bit-packed mask format (OCC_MASK_BITS, NEXT #4): every
kernel that writes masks (k_line's row / column / diagonal stores and its
per-pixel fallback, k_hard, k_tile for knight families, k_direct) sets
exactly the bits of the uint8 masks, padding bits stay 0, and the host
entry point moves the packed planes."""
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


def run(torch, D, views, fmt, path="auto"):
    from paper_2408_14050_b200.occ import Detector
    D = np.ascontiguousarray(D, np.float32)
    if D.ndim == 2:
        D = D[None]
    B, H, W = D.shape
    det = Detector(H, W, views, max_batch=B, path=path, mask_format=fmt)
    m = det.detect(torch.from_numpy(D).cuda())
    torch.cuda.synchronize()
    st = det.status()
    det.close()
    return m.cpu().numpy(), st


def check(torch, D, views, path="auto", oracle_frames=(0,)):
    from paper_2408_14050_b200.occ import unpack_masks
    u8, st8 = run(torch, D, views, "u8", path)
    pk, stp = run(torch, D, views, "bits", path)
    W = D.shape[-1]
    assert st8 == stp
    Wb = (W + 31) // 32
    assert pk.shape[-1] == Wb
    un = unpack_masks(pk, W)
    assert (un == u8).all()
    # padding bits of the last word are zero
    if W % 32:
        assert (pk.view(np.uint32)[..., -1] >> (W % 32) == 0).all()
    Ds = D if D.ndim == 3 else D[None]
    for f in oracle_frames:
        assert_same(un[f], oracle.detect(Ds[f], views), f"frame {f}")


def test_packed_c2_and_c3_crop(torch_cuda):
    check(torch_cuda, scenes.make_scene(2), scenes.VIEWS_3X3)
    check(torch_cuda, scenes.make_scene(3)[200:520, 300:901], scenes.VIEWS_3X3)


def test_packed_c4_crop_all_families(torch_cuda):
    # 5x5 array: knight families through k_tile, s = 2 pairs through k_line
    check(torch_cuda, scenes.make_scene(4)[1000:1300, 1500:1900], scenes.config_views(4))


@pytest.mark.parametrize("H,W", [(5, 7), (33, 65), (40, 130), (97, 131)])
def test_packed_small_and_ragged(torch_cuda, H, W):
    rng = scenes.SplitMix64(1401, H, W)
    D = np.stack([scenes.random_tiny_map(rng, H, W, m) for m in ("int", "half", "noisy", "uniform")])
    check(torch_cuda, D * 6.0, scenes.all_small_baselines(2) + [(3, 1), (0, -7)], oracle_frames=(0, 2))


def test_packed_direct_path_and_nonfinite(torch_cuda):
    D = scenes.make_batch(2, 3)
    D[1, 5, 5] = np.nan
    check(torch_cuda, D, scenes.VIEWS_3X3, path="direct")
    check(torch_cuda, D, scenes.VIEWS_3X3, path="auto")


def test_packed_host_entry_point(torch_cuda, monkeypatch):
    from paper_2408_14050_b200.occ import Detector, unpack_masks
    monkeypatch.setenv("OCC_CHUNK_MIB", "48")
    D = scenes.make_batch(5, 6)
    views = scenes.config_views(5)
    det = Detector(1080, 1920, views, max_batch=6, mask_format="bits")
    mh = det.detect_host(D)
    det.close()
    u8, _ = run(torch_cuda, D, views, "u8")
    assert mh.dtype == np.uint32 and mh.shape == (6, 8, 1080, 60)
    assert (unpack_masks(mh, 1920) == u8).all()
