"""Single-frame latency of C1-C3 per kernel path (auto / tiled / direct)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector  # noqa: E402
for cfg in (1, 2, 3, 4):
    D = scenes.make_scene(cfg)
    views = scenes.config_views(cfg)
    d = torch.from_numpy(D).cuda()[None]
    row = []
    for path in ("auto", "tiled", "direct"):
        det = Detector(D.shape[0], D.shape[1], views, path=path)
        out = det.detect(d)
        reps = 50 if cfg < 3 else 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(5):
            det.detect(d, out=out)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            det.detect(d, out=out)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{path} {e0.elapsed_time(e1) / reps * 1e3:.1f} us")
        det.close()
    print(f"C{cfg}:", ", ".join(row), flush=True)
