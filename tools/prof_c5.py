"""C5-style workload for profiling and A/B runs: F frames (default 32)
through occ_detect, REPS calls after one warm-up, with the SM clock sampled
during the timed calls and the per-kernel split of one more call (run under
ncu for per-kernel times)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector  # noqa: E402

F = int(os.environ.get("F", "32"))
reps = int(os.environ.get("REPS", "2"))
D = torch.from_numpy(scenes.make_batch(5, F)).cuda()
views = scenes.config_views(5)
det = Detector(1080, 1920, views, max_batch=F)
m = det.detect(D)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with ClockSampler(0) as clk:
    e0.record()
    for _ in range(reps):
        det.detect(D, out=m)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
mhz = statistics.median(clk.samples) if clk.samples else None
split = ""
if not os.environ.get("NO_SPLIT"):
    det.profile(True)
    det.detect(D, out=m)
    torch.cuda.synchronize()
    kt = det.profile_read()
    det.profile(False)
    split = " ".join(f"{k}={v[0]:.2f}" for k, v in kt.items() if v[1])
print(f"F={F} {ms:.3f} ms per call, {F * 1080 * 1920 * 8 / ms / 1e3:.0f} MPV/s, sm {mhz} MHz "
      f"{sorted(clk.reasons)} | {split}")
