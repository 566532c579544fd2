"""GPU parity of the median fusion kernel (occ_fuse_median, k_fuse.cu)
against the oracle.
Bit-exact fp32: every K of the unrolled kernels and the generic path, ragged
sizes (scalar tail path), ties, non-finite inputs, and the fused map driving
the detector (median of per-camera estimates -> occlusion masks)."""
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


def gpu_fuse(torch, st):
    from paper_2408_14050_b200.occ import fuse_median
    out = fuse_median(torch.from_numpy(np.ascontiguousarray(st, np.float32)).cuda())
    torch.cuda.synchronize()
    return out.cpu().numpy()


def same_f32(a, b, what):
    a = np.asarray(a, np.float32).view(np.uint32)
    b = np.asarray(b, np.float32).view(np.uint32)
    nan_a = (a & 0x7fffffff) > 0x7f800000
    nan_b = (b & 0x7fffffff) > 0x7f800000
    assert (nan_a == nan_b).all(), what
    bad = (~nan_a) & (a != b)
    assert not bad.any(), f"{what}: {int(bad.sum())} mismatches"


@pytest.mark.parametrize("K", list(range(1, 18)) + [24, 33, 64])
@pytest.mark.parametrize("n", [1, 3, 4, 1000, 4099])
def test_fuse_random(torch_cuda, K, n):
    rng = scenes.SplitMix64(1301, K, n)
    st = ((rng.uniform(K * n) - 0.3) * 80).astype(np.float32).reshape(K, n)
    same_f32(gpu_fuse(torch_cuda, st), oracle.fuse_median(st), f"K={K} n={n}")


def test_fuse_ties_and_nonfinite(torch_cuda):
    rng = scenes.SplitMix64(1302)
    for K in (2, 3, 8, 9):
        st = np.floor(rng.uniform(K * 4096) * 5).astype(np.float32).reshape(K, 4096)
        st[K // 2, 5] = np.nan
        st[0, 77] = np.inf
        st[K - 1, 4095] = -np.inf
        same_f32(gpu_fuse(torch_cuda, st), oracle.fuse_median(st), f"K={K}")


def test_fuse_then_detect(torch_cuda):
    # 8 per-camera estimates of a C3 crop (noise per estimate), fused on the GPU,
    # then detected: equal to the oracle's fusion + detection
    D = scenes.make_scene(3)[100:300, 500:900]
    rng = scenes.SplitMix64(1303)
    st = np.stack([D + 0.3 * rng.normal(D.size).reshape(D.shape).astype(np.float32) for _ in range(8)])
    st = st.astype(np.float32)
    fused_gpu = gpu_fuse(torch_cuda, st)
    fused_orc = oracle.fuse_median(st)
    same_f32(fused_gpu, fused_orc, "fused C3 crop")
    views = scenes.VIEWS_3X3
    g, _ = run_gpu(torch_cuda, fused_gpu, views)
    assert_same(g[0], oracle.detect(fused_orc, views), "masks of the fused map")


@pytest.mark.parametrize("K", [2, 3, 4, 5, 7, 8, 9, 16, 17])
def test_fuse_signed_zeros(torch_cuda, K):
    """-0 and +0 compare equal; the oracle's stable insertion sort keeps them in
    input order, so the median's zero sign is that of the zero a stable sort
    places in the middle.  Every pixel mixes -0, +0 and
    small integers; the check is bitwise."""
    rng = scenes.SplitMix64(1304, K)
    n = 8192
    u = rng.uniform(K * n).reshape(K, n)
    st = np.where(u < 0.3, -0.0, np.where(u < 0.6, 0.0, np.floor((u - 0.6) * 10) - 2.0)).astype(np.float32)
    assert (np.signbit(st) & (st == 0)).any() and ((~np.signbit(st)) & (st == 0)).any()
    same_f32(gpu_fuse(torch_cuda, st), oracle.fuse_median(st), f"K={K} signed zeros")
