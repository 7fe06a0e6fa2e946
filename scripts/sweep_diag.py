"""Diagnostics of the certified census sweep per level: undecided-bit rate,
exact samples, and the useful fraction of the (pixel, plane) slots the tiled
kernel iterates (a CTA walks the union of its 32x8 pixels' plane ranges)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_00821_b200 as pkg  # noqa: E402
from paper_2112_00821_b200 import Backend  # noqa: E402
import bench  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
scene, cfgkw, _ = bench.WORKLOADS[wl]
cfg = bench.make_config(pkg, **cfgkw)
for lvl in range(cfg.pyramid_levels):
    os.environ["FMVS_SWEEP_STATS"] = str(2 + lvl)
    b = Backend(os.environ["FMVS_LIB"], "fmvs_") if os.environ.get("FMVS_LIB") else Backend.b200()
    frames = bench.render_frames(b, scene, scene.get("views", 5))
    b.estimate_bundle(frames, cfg)
    out = (C.c_uint64 * 8)()
    b._check(b.fn["ctx_sweep_stats"](b.ctx, out))
    ev, unsure_ev, unsure_bits, exact_views, it_run, _, items, useful = list(out)
    print(f"level {lvl}: view-evals {ev}  with-undecided {100.0*unsure_ev/max(ev,1):.2f}%  undecided bits "
          f"{100.0*unsure_bits/max(ev*24,1):.3f}%  exact views {exact_views}  exact samples {items}")
    print(f"   tile-plane iterations {it_run}; useful (pixel, plane) slots {useful} of {256*it_run} "
          f"({100.0*useful/max(256*it_run,1):.1f}%)")
    b.close()
