"""GPU parity of the knight baselines (2, +-1), (1, +-2) through the sheared
frames (k_shear + k_sweep<SHEAR> + k_hard<SHEAR>): digital
lines of slope 1/2 (reading Q8) on concurrent streams.
The host-buffer entry point (its own copy streams), a captured CUDA graph
(the fork / join of the family streams inside the capture), both masks
formats and odd image sizes (the sheared frame's padding) against the oracle.
"""
import numpy as np
import pytest

import oracle
from paper_2408_14050_b200 import scenes
from test_gpu_parity import assert_same, run_gpu, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu

KNIGHTS = [(2, 1), (-2, -1), (2, -1), (-2, 1), (1, 2), (-1, -2), (1, -2), (-1, 2)]


def test_knights_only(torch_cuda):
    # only sheared families: no main sweep units at all
    D = scenes.make_scene(4)[700:890, 900:1210].copy()
    g, st = run_gpu(torch_cuda, D, KNIGHTS)
    assert st == [0]
    assert_same(g[0], oracle.detect(D, KNIGHTS), "knights only")


@pytest.mark.parametrize("H,W", [(131, 257), (97, 301), (260, 130)])
def test_knights_odd_sizes(torch_cuda, H, W):
    rng = scenes.SplitMix64(4242, H, W)
    D = (scenes.random_tiny_map(rng, H, W, "int") * 6.0).astype(np.float32)
    views = KNIGHTS + [(1, 0), (0, -1)]
    g, _ = run_gpu(torch_cuda, D, views)
    assert_same(g[0], oracle.detect(D, views), f"{H}x{W}")


def test_knights_host_entry(torch_cuda):
    from paper_2408_14050_b200.occ import Detector
    D = np.stack([scenes.make_scene(4, 0, f)[1000:1200, 1500:1800] for f in range(3)])
    views = scenes.VIEWS_5X5
    det = Detector(200, 300, views, max_batch=3)
    mh = det.detect_host(D)
    det.close()
    for f in range(3):
        assert_same(mh[f], oracle.detect(D[f], views), f"host frame {f}")


@pytest.mark.parametrize("fmt", ["u8", "bits"])
def test_knights_graph_capture(torch_cuda, fmt):
    torch = torch_cuda
    from paper_2408_14050_b200.occ import Detector, unpack_masks
    D = scenes.make_scene(4)[400:592, 2000:2320].copy()
    views = scenes.VIEWS_5X5
    det = Detector(192, 320, views, max_batch=1, mask_format=fmt)
    d = torch.from_numpy(D[None]).cuda()
    ref = det.detect(d).clone()
    out = torch.zeros_like(ref)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        det.detect(d, out=out)               # warm-up on the capture stream
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        det.detect(d, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    m = out.cpu().numpy()
    if fmt == "bits":
        m = unpack_masks(m.view(np.uint32), 320)
    assert_same(m[0], oracle.detect(D, views), f"graph {fmt}")
    det.close()
