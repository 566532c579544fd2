"""C5-style workload for profiling: F frames (default 32) through occ_detect,
`reps` calls after one warm-up (run under ncu for per-kernel times)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2408_14050_b200 import scenes
from paper_2408_14050_b200.occ import Detector

F = int(os.environ.get("F", "32"))
reps = int(os.environ.get("REPS", "2"))
D = torch.from_numpy(scenes.make_batch(5, F)).cuda()
views = scenes.config_views(5)
det = Detector(1080, 1920, views, max_batch=F)
m = det.detect(D)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    det.detect(D, out=m)
e1.record()
torch.cuda.synchronize()
print(f"F={F} {e0.elapsed_time(e1) / reps:.3f} ms per call, {F * 1080 * 1920 * 8 / (e0.elapsed_time(e1) / reps) / 1e3:.0f} MPV/s")
