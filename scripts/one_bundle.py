"""Runs N bundles of a bench workload through the host API (profiling target for ncu)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_00821_b200 as pkg
from paper_2112_00821_b200 import Backend
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = sys.argv[2] if len(sys.argv) > 2 else "c2"
b = Backend.b200()
scene, cfgkw, _ = bench.WORKLOADS[wl]
frames = bench.render_frames(b, scene, scene.get("views", 5))
cfg = bench.make_config(pkg, **cfgkw)
for _ in range(n):
    b.estimate_bundle(frames, cfg)
print(b.level_stats())
