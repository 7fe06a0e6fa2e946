"""Diagnostics: certified-census fallback rate and per-kernel split on C2."""
import ctypes as C
import os
import sys
os.environ["FMVS_SWEEP_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_00821_b200 as pkg
from paper_2112_00821_b200 import Backend
import bench

b = Backend(os.environ["FMVS_LIB"], "fmvs_") if os.environ.get("FMVS_LIB") else Backend.b200()
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
scene, cfgkw, _ = bench.WORKLOADS[wl]
frames = bench.render_frames(b, scene, scene.get("views", 5))
cfg = bench.make_config(pkg, **cfgkw)
b.estimate_bundle(frames, cfg)
out = (C.c_uint64 * 8)()
b._check(b.fn["ctx_sweep_stats"](b.ctx, out))
ev, unsure_ev, unsure_bits, exact_views, it_run, it_skip, items, _ = list(out)
print(f"view-evals {ev}  with-undecided {unsure_ev} ({100.0*unsure_ev/max(ev,1):.2f}%)  "
      f"undecided bits {unsure_bits} ({100.0*unsure_bits/max(ev*24,1):.3f}% of bits)  exact views {exact_views}")
print(f"tile-plane iterations run {it_run} skipped {it_skip}; hypothesis-views per run iteration "
      f"{ev / max(it_run, 1):.1f} (of 256 x views); exact samples {items}")
print(b.level_stats())
