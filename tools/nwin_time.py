"""Time the finite-N kernel (k_nwin) vs the N = infinity path on the C5
workload (device buffers, occ_profile device times)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import numpy as np
import torch

from paper_2408_14050_b200 import scenes
from paper_2408_14050_b200.occ import Detector

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 64
Ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 8]
D = torch.from_numpy(scenes.make_batch(5, frames)).cuda()
views = scenes.config_views(5)
for N in Ns:
    det = Detector(1080, 1920, views, max_batch=frames, neighbors=N, mask_format="bits")
    out = None
    for _ in range(2):
        out = det.detect(D, out)
    torch.cuda.synchronize()
    det.profile(True)
    t = time.time()
    for _ in range(3):
        out = det.detect(D, out)
    torch.cuda.synchronize()
    wall = (time.time() - t) / 3
    prof = det.profile_read()
    det.profile(False)
    print(f"N={N}: wall {wall * 1e3:.2f} ms/step ({frames} frames) "
          f"-> {frames * 1920 * 1080 * len(views) / wall / 1e6:.0f} MPV/s; kernels "
          + ", ".join(f"{k} {v[0] / 3:.2f} ms" for k, v in prof.items() if v[1]), flush=True)
    det.close()
