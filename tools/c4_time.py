"""C4 (2 frames, 24 views) device time per call and per-kernel split."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector  # noqa: E402
D = np.stack([scenes.make_scene(4, 0, f) for f in range(2)])
views = scenes.config_views(4)
d = torch.from_numpy(D).cuda()
det = Detector(D.shape[1], D.shape[2], views, max_batch=2)
out = det.detect(d)
det.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    det.detect(d, out=out)
e1.record()
torch.cuda.synchronize()
kt = det.profile_read()
print(f"C4 2 frames: {e0.elapsed_time(e1) / 5:.3f} ms;", {k: round(v[0] / 5, 3) for k, v in kt.items() if v[1]})
