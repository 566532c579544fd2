"""Run one view pair (rows/cols/diag/anti) of C3 frames repeatedly (profiling helper)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector  # noqa: E402

FAM = {"rows": [(1, 0), (-1, 0)], "cols": [(0, 1), (0, -1)], "diag": [(1, 1), (-1, -1)],
       "anti": [(1, -1), (-1, 1)], "all": scenes.VIEWS_3X3}
fam = sys.argv[1] if len(sys.argv) > 1 else "rows"
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 4
D = torch.from_numpy(scenes.make_batch(3, nf)).cuda()
det = Detector(D.shape[1], D.shape[2], FAM[fam], max_batch=nf)
for _ in range(3):
    det.detect(D)
torch.cuda.synchronize()
print("ok", fam, nf)
