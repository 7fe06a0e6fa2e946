"""Per-level hypothesis-count distribution of a bench workload and, per SGM
direction class, how many scanlines contain a pixel wider than a cap."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2112_00821_b200 as pkg  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
b = pkg.Backend.b200()
scene, cfgkw, _ = bench.WORKLOADS[wl]
frames = bench.render_frames(b, scene, scene.get("views", 5))
cfg = bench.make_config(pkg, **cfgkw)
for lvl in range(cfg.pyramid_levels):
    cap = b.estimate_bundle_captured(frames, cfg, level=lvl)
    hh, ww = cap["depth_raw"].shape
    cnt = cap["count"].reshape(hh, ww)
    print(f"level {lvl}: shape {cnt.shape} mean {cnt.mean():.2f} max {cnt.max()} "
          f"pct>16 {100*(cnt>16).mean():.3f} pct>32 {100*(cnt>32).mean():.3f} pct>64 {100*(cnt>64).mean():.4f}")
    for capv in (16, 32, 64):
        wide = cnt > capv
        rows = wide.any(axis=1).mean()
        cols = wide.any(axis=0).mean()
        ys, xs = np.nonzero(wide)
        d1 = len(np.unique(xs - ys)) / (hh + ww - 1)
        print(f"   cap {capv}: rows with a wide pixel {100*rows:.1f}%  cols {100*cols:.1f}%  diagonals {100*d1:.1f}%")
    bc = np.bincount(np.minimum(cnt.ravel(), 40), minlength=41)
    print("   count histogram (0..39, >=40):", " ".join(f"{i}:{v}" for i, v in enumerate(bc) if v))
