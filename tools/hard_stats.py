import os, sys, ctypes
sys.path.insert(0, os.getcwd())
os.environ["OCC_LIB"] = os.path.join(os.getcwd(), "paper_2408_14050_b200/libocc_hst.so")
import torch
from paper_2408_14050_b200 import scenes
from paper_2408_14050_b200.occ import Detector, lib
D = torch.from_numpy(scenes.make_batch(5, 16)).cuda()
det = Detector(1080, 1920, scenes.config_views(5), max_batch=16)
det.detect(D); torch.cuda.synchronize()
L = lib(); L.occ_debug_hard_stats.argtypes = [ctypes.c_void_p]
out = (ctypes.c_ulonglong * 8)()
L.occ_debug_hard_stats(out)
n, hits, scanned, jmsum = out[0], out[1], out[2], out[3]
pv = 16 * 1920 * 1080 * 8
print(f"entries {n} ({n/pv*100:.2f}% of pixel-views), hits {hits} ({hits/max(n,1)*100:.1f}%), avg scan range {scanned/max(n,1):.1f}, avg dcov {jmsum/max(n,1):.1f}")
