"""bench.py h-sweep leg alone (32 C5 frames, scaled to each target h)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())

if __name__ == "__main__":      # (the leg spawns scene-generation workers)
    import bench
    from paper_2408_14050_b200 import scenes
    fr = bench.make_frames(32, 0)
    print(json.dumps(bench.h_sweep_leg(fr, scenes.config_views(5), 6456.8)))
