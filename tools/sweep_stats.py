"""Event counters of k_sweep (SWEEP_STATS build) on C5 frames.
Run: OCC_DEFINES=-DSWEEP_STATS python tools/sweep_stats.py [frames]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14050_b200 import build  # noqa: E402
os.environ["OCC_LIB"] = build.build()
import torch  # noqa: E402
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector, lib  # noqa: E402

L = lib()
L.occ_debug_line_stats.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_ulonglong)]
names = ["positions", "survP", "survN", "hit1P", "hit1N", "hit2P", "hit2N", "queuedP", "queuedN", "rounds",
         "nearP", "nearN", "survblocks", "blocks"]
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 4
D = torch.from_numpy(scenes.make_batch(5, nf)).cuda()
H, W = D.shape[1:]
for fam, views in [("rows", [(1, 0), (-1, 0)]), ("cols", [(0, 1), (0, -1)]),
                   ("diag", [(1, 1), (-1, -1)]), ("anti", [(1, -1), (-1, 1)]), ("all", scenes.VIEWS_3X3)]:
    det = Detector(H, W, views, max_batch=nf)
    det.detect(D)
    torch.cuda.synchronize()
    L.occ_debug_line_stats(det._h, 1, None)
    det.detect(D)
    out = (ctypes.c_ulonglong * (16 + 65536 + 4 * 32768))()
    L.occ_debug_line_stats(det._h, 0, out)
    v = list(out)[:14]
    pos = max(1, v[0])
    print(f"{fam:5s} " + " ".join(f"{n}={x / pos:.5f}" if i else f"{n}={x}" for i, (n, x) in enumerate(zip(names, v))))
    det.close()
