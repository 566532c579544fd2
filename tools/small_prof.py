"""Launch list of one small-config detect (C1 or C2) for ncu."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector  # noqa: E402
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
D = scenes.make_scene(cfg)
det = Detector(D.shape[0], D.shape[1], scenes.config_views(cfg))
d = torch.from_numpy(D).cuda()[None]
for _ in range(3):
    det.detect(d)
torch.cuda.synchronize()
