"""GPU parity of real-valued baseline directions (occ_create_dirs, NEXT #2,
reading Q23) against the oracle's orc_detect_dirs, bit-exact: angle 0 equal
to the grid baselines, random angles and lengths on layered and tiny maps
(N = infinity and finite N), a perturbed 3x3 "calibrated" array on a C3
crop, long windows (global-scratch launch), both mask formats, small
max_scan caps and non-finite frames."""
import math

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


def run(torch, D, dirs, N=0, fmt="u8", host=False, **kw):
    from paper_2408_14050_b200.occ import Detector, unpack_masks
    D = np.ascontiguousarray(D, np.float32)
    if D.ndim == 2:
        D = D[None]
    B, H, W = D.shape
    det = Detector(H, W, directions=dirs, max_batch=B, mask_format=fmt, neighbors=N, **kw)
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


def calibrated(rng, n=8, jitter=0.05):
    """A perturbed ring of n peripheral cameras (angles k 2pi/n + noise,
    lengths 1 or sqrt(2) times 1 +- 5 %)."""
    out = []
    for k in range(n):
        u = rng.uniform(2)
        a = 2 * math.pi * k / n + jitter * (2 * u[0] - 1)
        r = (math.sqrt(2) if k % 2 else 1.0) * (1 + jitter * (2 * u[1] - 1))
        out.append((a, r))
    return out


def test_angle_zero_equals_grid(torch_cuda):
    from test_gpu_parity import run_gpu
    rng = scenes.SplitMix64(6101)
    D = np.stack([layered(rng, 64, 96, 10, 1.0, 20.0, 0.25) for _ in range(2)])
    a, _ = run(torch_cuda, D, [(0.0, 1.0), (0.0, 2.0)])
    b, _ = run_gpu(torch_cuda, D, [(1, 0), (2, 0)])
    assert (a == b).all()


@pytest.mark.parametrize("N", [0, 8])
@pytest.mark.parametrize("H,W", [(70, 90), (97, 131), (33, 200)])
def test_dirs_layered(torch_cuda, N, H, W):
    rng = scenes.SplitMix64(6102, H, W, N)
    dirs = calibrated(rng) + [(0.3, 1.0), (2.2, 1.7), (4.0, 0.6)]
    D = np.stack([layered(rng, H, W, 12, 1.0, 25.0, 0.25 * f) for f in range(2)])
    g, st = run(torch_cuda, D, dirs, N)
    assert st == [0, 0]
    for f in range(2):
        assert_same(g[f], oracle.detect_dirs(D[f], dirs, neighbors=N), f"{H}x{W} N={N} frame {f}")


@pytest.mark.parametrize("chunk", range(3))
def test_dirs_tiny_maps(torch_cuda, chunk):
    rng = scenes.SplitMix64(6103, chunk)
    for it in range(10):
        H, W = rng.randint(3, 24), rng.randint(3, 24)
        D = scenes.random_tiny_map(rng, H, W, MODES[it % 4])
        u = rng.uniform(6)
        dirs = [(2 * math.pi * u[k], 0.3 + 3.0 * u[k + 3]) for k in range(3)]
        N = [0, 2, 8, 0][it % 4]
        kw = {} if it % 3 else dict(t_dist=1.0, t_disp=0.25)
        g, _ = run(torch_cuda, D, dirs, N, **kw)
        assert_same(g[0], oracle.detect_dirs(D, dirs, neighbors=N, **kw), f"chunk {chunk} it {it}")


def test_dirs_c3_crop_calibrated(torch_cuda):
    rng = scenes.SplitMix64(6104)
    dirs = calibrated(rng)
    D = np.ascontiguousarray(scenes.make_scene(3)[300:620, 500:1000])
    g, _ = run(torch_cuda, D, dirs, fmt="bits")
    o = oracle.detect_dirs(D, dirs)
    for i, d in enumerate(dirs):
        assert_same(g[0, i], o[i], f"C3 crop dir {d}")


def test_dirs_long_windows(torch_cuda):
    # length 4.5 over disparities [1, 40]: h ~ 175 > 159 -> global scratch
    rng = scenes.SplitMix64(6105)
    D = layered(rng, 40, 300, 10, 1.0, 40.0, 0.25)
    dirs = [(0.1, 4.5), (3.3, 4.5), (1.2, 1.0)]
    for N in (0, 8):
        g, _ = run(torch_cuda, D, dirs, N)
        assert_same(g[0], oracle.detect_dirs(D, dirs, neighbors=N), f"long N={N}")


def test_dirs_caps_nonfinite_host(torch_cuda):
    rng = scenes.SplitMix64(6106)
    D = np.stack([layered(rng, 50, 70, 8, 1.0, 20.0, 0.25) for _ in range(3)])
    D[1, 3, 3] = np.nan
    dirs = calibrated(rng, 6)
    for cap in (1, 2, 9):
        g, st = run(torch_cuda, D, dirs, max_scan=cap)
        assert st[1] != 0 and g[1].sum() == 0
        assert_same(g[0], oracle.detect_dirs(D[0], dirs, max_scan=cap), f"cap {cap}")
    h, _ = run(torch_cuda, D, dirs, host=True)
    d, _ = run(torch_cuda, D, dirs)
    assert (h == d).all()


def test_dirs_argument_validation(torch_cuda):
    from paper_2408_14050_b200.occ import Detector, OccError
    for bad in ([(float("nan"), 1.0)], [(0.0, 0.0)], [(0.0, 8.5)]):
        with pytest.raises(OccError):
            Detector(16, 16, directions=bad)
    with pytest.raises(ValueError):
        Detector(16, 16)


def test_dirs_full_c5_frames_bench_launch(torch_cuda):
    # the launch configuration bench.py's directions leg times: one call over a
    # batch of C5 frames with the bench's 8 calibrated directions; sampled
    # whole frames vs the oracle
    import bench
    dirs = bench.calibrated_dirs()
    D = scenes.make_batch(5, 4)
    g, st = run(torch_cuda, D, dirs, fmt="bits")
    assert st == [0] * 4
    for f in (0, 3):
        o = oracle.detect_dirs(D[f], dirs)
        for i, d in enumerate(dirs):
            assert_same(g[f, i], o[i], f"C5 frame {f} dir {d}")
