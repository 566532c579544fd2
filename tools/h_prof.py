"""Per-kernel device time (occ_profile) of 8 C5 frames scaled to several h."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector  # noqa: E402

fr = bench.make_frames(8, 0)
views = scenes.config_views(5)
det = Detector(fr.shape[1], fr.shape[2], views, max_batch=8)
for ht in [65, 150, 300, 600]:
    d = torch.from_numpy(scenes.scale_disparity(fr, ht / 65.0)).cuda()
    m = det.detect(d)
    torch.cuda.synchronize()
    det.profile(True)
    det.detect(d, out=m)
    torch.cuda.synchronize()
    kt = det.profile_read()
    det.profile(False)
    print(ht, det.frame_info(0)[2][:2], {k: round(v[0], 3) for k, v in kt.items() if v[1]}, int(m.sum()))
