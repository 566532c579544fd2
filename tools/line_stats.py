"""Event statistics of the line-sweep kernel on C3 frames, per line family
(debug tool; uses the non-public occ_debug_line_stats entry point)."""
import ctypes
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14050_b200 import scenes  # noqa: E402
from paper_2408_14050_b200.occ import Detector, lib  # noqa: E402

L = lib()
L.occ_debug_line_stats.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_ulonglong)]
names = ["survP", "survN", "stage1_hits", "hard", "exh_found", "exh_steps", "global_probes",
         "blocks(x32)", "direct_units", "resolve_iters(x32)"]
names2 = ["q_overflow", "q_tot", "q_n", "after_stage1"]
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 4
D = torch.from_numpy(scenes.make_batch(3, nf)).cuda()
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
    pv = nf * H * W * len(views)
    vals = list(out)[:10]
    print(fam, " ".join(f"{n}={v / pv:.5f}" if i not in (7, 9) else f"{n}={v / 32 / pv:.5f}"
                        for i, (n, v) in enumerate(zip(names, vals))))
    print("   raw:", {n: int(v) for n, v in zip(names2, list(out)[10:14])}, "steps", int(out[5]))
    allv = np.array(list(out)[16:16 + 65536], dtype=np.uint64)
    phs = np.array(list(out)[16 + 65536:16 + 65536 + 4 * 32768], dtype=np.float64).reshape(-1, 4)
    print("   phase totals / CTA-cycles: resolve %.3f flush %.3f pass0 %.3f" % tuple(
        phs[:, i].sum() / max(1.0, float(allv[:32768].astype(np.float64).sum())) for i in range(3)))
    cyc = allv[:32768].astype(np.float64)
    info = allv[32768:]
    top = np.argsort(-cyc)[:6]
    for t in top:
        if cyc[t] <= 0: continue
        iv = int(info[t])
        ph = [int(out[16 + 2 * 32768 + 4 * t + i]) for i in range(3)]
        print("     slow CTA %d: %.0f cyc kind %d len %d l0 %d t0 %d | resolve %d flush %d pass0 %d" % (
              t, cyc[t], iv >> 60, (iv >> 40) & 0xfffff, ((iv >> 20) & 0xfffff) - 40000, (iv & 0xfffff) - 40000,
              ph[0], ph[1], ph[2]))
    cyc = cyc[cyc > 0]
    if len(cyc):
        print("   CTA cycles: n=%d mean=%.0f p50=%.0f p90=%.0f p99=%.0f max=%.0f sum/148=%.0f" % (
            len(cyc), cyc.mean(), np.percentile(cyc, 50), np.percentile(cyc, 90), np.percentile(cyc, 99),
            cyc.max(), cyc.sum() / 148))
    # timing
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3):
        det.detect(D)
    torch.cuda.synchronize()
    print(f"   {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms per call of {nf} frames")
    det.close()
