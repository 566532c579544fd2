"""Small detections for compute-sanitizer runs (one tool per gpurun call):
the line sweep on a C2 crop and a noisy C3 crop (uint8 and bit-packed masks,
both views of every family), a forced far-partner queue overflow
(OCC_GQ_CAP=37: straddling reservations, in-warp fallback, k_hard), the
knight Eq. 2 overflow repro, a C4 crop with the 5x5 array (sheared knight
families), crops at h ~ 5 and ~ 300, and the median fusion; every output is
checked against the oracle.  Usage: compute-sanitizer --tool X python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_2408_14050_b200 import scenes
from paper_2408_14050_b200.occ import Detector, fuse_median, unpack_masks


def run(D, views, what, **kw):
    D = np.ascontiguousarray(D, np.float32)
    if D.ndim == 2:
        D = D[None]
    B, H, W = D.shape
    for fmt in ("u8", "bits"):
        det = Detector(H, W, views, max_batch=B, mask_format=fmt, **kw)
        m = det.detect(torch.from_numpy(D).cuda())
        torch.cuda.synchronize()
        g = m.cpu().numpy()
        if fmt == "bits":
            g = unpack_masks(g.view(np.uint32), W)
        for f in range(B):
            o = oracle.detect(D[f], views, **kw)
            assert (g[f] == o).all(), f"{what} {fmt} frame {f}"
        det.close()
    print("ok", what, flush=True)


run(scenes.make_scene(2)[100:228, 200:392], scenes.VIEWS_3X3, "C2 crop")
run(np.stack([scenes.make_scene(3)[300:428, 700:956], scenes.make_scene(3, frame=1)[0:128, 0:256]]),
    scenes.VIEWS_3X3, "C3 crops")
os.environ["OCC_GQ_CAP"] = "37"
run(scenes.make_scene(3)[200:328, 600:856], scenes.VIEWS_3X3, "C3 crop, queue capacity 37")
del os.environ["OCC_GQ_CAP"]
Dk = np.zeros((64, 160), np.float32)
Dk[:, 21:] = 3e38
Dk[3:, :21] = -3e38
Dk[2, 20] = 1e38
Dk[0, 17] = Dk[0, 18] = Dk[1, 17] = 1.0
run(Dk, scenes.VIEWS_5X5, "knight overflow repro", max_scan=150)
# knight baselines through the sheared frames (both majors), small and large h
run(scenes.make_scene(4)[1000:1160, 1500:1820], scenes.VIEWS_5X5, "C4 crop, 5x5 array (sheared knights)")
D3 = scenes.make_scene(3)[300:460, 700:1020].astype(np.float64)
R = float(D3.max() - D3.min())
run(scenes.scale_disparity(D3, 5.0 / R), scenes.VIEWS_3X3, "C3 crop at h ~ 5 (k_sweep_small)")
run(scenes.scale_disparity(D3, 300.0 / R), scenes.VIEWS_3X3, "C3 crop at h ~ 300")
rng = scenes.SplitMix64(77)
st = ((rng.uniform(8 * 4099) - 0.3) * 80).astype(np.float32).reshape(8, 4099)
out = fuse_median(torch.from_numpy(st).cuda()).cpu().numpy()
assert (out.view(np.uint32) == oracle.fuse_median(st).view(np.uint32)).all()
print("ok fuse", flush=True)
