"""Host-side cost of enqueueing one C2 bundle (planning + launches), measured
without synchronising (the launch queue holds ~20 bundles)."""
import ctypes as C
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_00821_b200 as pkg
from paper_2112_00821_b200 import Backend, _abi
import bench

b = Backend.b200()
scene, cfgkw, _ = bench.WORKLOADS["c2"]
frames = bench.render_frames(b, scene, 5)
cfg = bench.make_config(pkg, **cfgkw).to_c()
h, w = frames[0].image.shape
d = torch.from_numpy(np.stack([f.image for f in frames])).cuda()
arr = (_abi.View_c * 5)()
for k in range(5):
    arr[k].image = d[k].data_ptr()
    arr[k].intrinsics = frames[k].intrinsics.to_c()
    arr[k].pose = frames[k].pose.to_c()
o = [torch.empty(w * h * 5, dtype=torch.float32, device="cuda") for _ in range(1)]
fn = b.fn["estimate_bundle_device"]
for _ in range(3):
    fn(b.ctx, arr, 5, C.byref(cfg), o[0].data_ptr(), o[0].data_ptr() + 4 * w * h, o[0].data_ptr() + 16 * w * h)
b._check(b.fn["ctx_synchronize"](b.ctx))
ts = []
for _ in range(8):
    t0 = time.perf_counter()
    fn(b.ctx, arr, 5, C.byref(cfg), o[0].data_ptr(), o[0].data_ptr() + 4 * w * h, o[0].data_ptr() + 16 * w * h)
    ts.append(time.perf_counter() - t0)
b._check(b.fn["ctx_synchronize"](b.ctx))
print("host enqueue ms per bundle:", [round(1e3 * t, 3) for t in ts])
