"""Per-call latency of one small config (C2 / C3: one frame) and its kernel
split (occ_profile), for tuning the single-frame path.  Usage: small_time.py cfg"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector  # noqa: E402
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
D = scenes.make_scene(cfg)
det = Detector(D.shape[0], D.shape[1], scenes.config_views(cfg))
d = torch.from_numpy(D).cuda()[None]
m = det.detect(d)
for _ in range(5):
    det.detect(d, out=m)
torch.cuda.synchronize()
n = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    det.detect(d, out=m)
e1.record()
torch.cuda.synchronize()
det.profile(True)
for _ in range(n):
    det.detect(d, out=m)
torch.cuda.synchronize()
kt = det.profile_read()
det.profile(False)
print(f"C{cfg} {e0.elapsed_time(e1) / n * 1e3:.1f} us/call;",
      " ".join(f"{k}={v[0] / n * 1e3:.1f}us" for k, v in kt.items() if v[1]))
