#!/usr/bin/env python3
"""Benchmark of the per-frame depth+normal path (estimate_bundle) on B200.

Contract (see the task's bench.py spec): `python bench.py --gpus N --steps K
--warmup W [--impl b200|reference]`; one process per GPU under torchrun for
N>1; rank 0 prints ONE JSON line.

Workload (BASELINE.json configs[1], SURVEY.md §8d "C2"): slanted_scene
1920x1080, f=1920, plane tilted 30 deg at depth 10, 5 views on a lateral
track (step 0.59), depth range 4:40, 3 pyramid levels, max_planes 128 at the
coarsest level, census 5x5, SGM Pi-sn over 8 paths, normals + confidence.
A step = one estimate_bundle of one bundle. Each rank runs its own stream of
bundles (independent bundles: weak scaling, no collective on the data path).

value : maps/s of the whole job, inputs resident in HBM, device-timed per
        step with CUDA events on the library's stream, L2 flushed (256 MiB
        memset) before every timed step; max over ranks.
e2e   : the same metric through the public C ABI (fmvs_estimate_bundle) with
        pinned HOST buffers: 5 images H2D + depth/normals/confidence D2H
        inside the timed region (wall clock around the blocking calls).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Full-HD depth+normal maps/sec and MDE/s per GPU, 1/2/4/8 B200 vs CPU"

WORKLOADS = {
    # name: (scene kwargs, config kwargs, description)
    "c2": (dict(kind="slanted", width=1920, height=1080, focal=1920.0, depth=10.0, tilt=30.0,
                step=0.59, texture=0.1),
           dict(d_min=4.0, d_max=40.0, levels=3, max_planes=128, cost="census5", variant="sn", paths=8),
           "C2: slanted_scene 1920x1080 f=1920 tilt 30deg depth 10, 5 views lateral step 0.59, "
           "range 4:40, 3 levels, max_planes 128 (coarsest), census 5x5, SGM pi-sn 8 paths, "
           "normals+confidence"),
    "c1": (dict(kind="fronto", width=640, height=480, focal=640.0, depth=10.0, tilt=0.0, step=1.82,
                texture=0.1, views=3),
           dict(d_min=8.0, d_max=14.0, levels=1, max_planes=64, cost="census5", variant="plane", paths=8),
           "C1: fronto_scene 640x480, 3 views, 1 level, 64 planes, census 5x5, SGM pi 8 paths"),
}


def make_config(pkg, d_min, d_max, levels, max_planes, cost, variant, paths):
    kinds = {"census5": (pkg.CostKind.CensusHamming, 5, 5), "ncc5": (pkg.CostKind.NccTruncated, 5, 5)}
    var = {"plane": pkg.SgmVariant.Plane, "sn": pkg.SgmVariant.SurfaceNormal,
           "pg": pkg.SgmVariant.PathGradient}[variant]
    k, ww, wh = kinds[cost]
    return pkg.PipelineConfig(d_min, d_max, pyramid_levels=levels, max_planes=max_planes,
                              sgm=pkg.SgmConfig(variant=var, paths=paths),
                              cost=pkg.CostFunctionSpec(k, ww, wh))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def render_frames(b200, scene, frames):
    """Renders a lateral track of `frames` views on the device (render.cpp)."""
    bundle, _, _ = b200.render_plane_scene(
        scene["kind"], scene["width"], scene["height"], scene["focal"], scene["depth"], frames,
        scene["step"], seed=1, tilt_deg=scene["tilt"], texture_scale=scene["texture"])
    return bundle


def alg_bytes(stage, stats, n_views, paths):
    """Algorithmic HBM bytes of one stage summed over levels."""
    tot = 0
    for lv in stats:
        px = lv["width"] * lv["height"]
        e = lv["entries"]
        if stage.startswith("sgm"):
            if (stage == "sgm_l0") != (lv is stats[0]):
                continue
            tot += e * (2 * paths + 4) + px * paths * 9
        elif stage.startswith("sweep"):
            if (stage == "sweep_l0") != (lv is stats[0]):
                continue
            tot += e * 2 + px * (8 + n_views)
    return tot


def run_b200(args, rank, world, device):
    import torch
    import paper_2112_00821_b200 as pkg
    from paper_2112_00821_b200 import Backend

    scene, cfgkw, desc = WORKLOADS[args.workload]
    views = scene.get("views", 5)
    torch.cuda.set_device(device)
    b200 = Backend.b200(device)
    cfg = make_config(pkg, **cfgkw)
    ring = args.ring
    frames = render_frames(b200, scene, ring + views - 1)
    h, w = frames[0].image.shape
    px = w * h
    # device-resident frames + outputs
    d_frames = torch.from_numpy(np.stack([f.image for f in frames])).to(f"cuda:{device}")
    d_depth = torch.empty((h, w), dtype=torch.float32, device=f"cuda:{device}")
    d_norm = torch.empty((h, w, 3), dtype=torch.float32, device=f"cuda:{device}")
    d_conf = torch.empty((h, w), dtype=torch.float32, device=f"cuda:{device}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")
    stream = torch.cuda.ExternalStream(b200.fn["ctx_stream"](b200.ctx), device=f"cuda:{device}")

    from paper_2112_00821_b200 import _abi
    from paper_2112_00821_b200.fassmvs import _views_c

    def views_for(i, dev=True):
        s = i % ring
        arr = (_abi.View_c * views)()
        for k in range(views):
            f = frames[s + k]
            arr[k].image = d_frames[s + k].data_ptr() if dev else f.image.ctypes.data
            arr[k].intrinsics = f.intrinsics.to_c()
            arr[k].pose = f.pose.to_c()
        return arr

    ccfg = cfg.to_c()
    vlist = [views_for(i) for i in range(ring)]

    def step(i):
        rc = b200.fn["estimate_bundle_device"](b200.ctx, vlist[i % ring], views, C.byref(ccfg),
                                               d_depth.data_ptr(), d_norm.data_ptr(), d_conf.data_ptr())
        if rc != 0:
            b200._check(rc)

    # warmup
    for i in range(args.warmup):
        step(i)
    b200._check(b200.fn["ctx_synchronize"](b200.ctx))
    stats = b200.level_stats()
    launches_per_step = b200.last_launch_count()

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(device) as clocks:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()               # L2 flush, outside the timed events
                evs[i][0].record(stream)
            step(args.warmup + i)
            with torch.cuda.stream(stream):
                evs[i][1].record(stream)
        b200._check(b200.fn["ctx_synchronize"](b200.ctx))
        torch.cuda.synchronize(device)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    maps_per_s = world * args.steps * 1000.0 / total_ms
    entries = sum(lv["entries"] for lv in stats)

    # ---- per-stage CUDA-event timing pass (roofline of the dominant kernel)
    b200.fn["ctx_set_timing"](b200.ctx, 1)
    b200.fn["ctx_stage_reset"](b200.ctx)
    nprof = max(3, min(args.steps, 8))
    for i in range(nprof):
        with torch.cuda.stream(stream):
            flush.zero_()
        step(i)
        b200._check(b200.fn["ctx_synchronize"](b200.ctx))
    b200.fn["ctx_set_timing"](b200.ctx, 0)
    stages = {}
    for i in range(b200.fn["ctx_stage_count"](b200.ctx)):
        ms, calls = C.c_double(), C.c_int64()
        b200.fn["ctx_stage_time"](b200.ctx, i, C.byref(ms), C.byref(calls))
        name = b200.fn["ctx_stage_name"](b200.ctx, i).decode()
        stages[name] = {"ms_per_step": ms.value / nprof, "launches_per_step": calls.value / nprof}
    peak, peak_src = peaks()
    for name, st in stages.items():
        b = alg_bytes(name, stats, views, cfg.sgm.paths)
        st["alg_bytes"] = b
        st["gbs"] = b / (st["ms_per_step"] * 1e6) if b and st["ms_per_step"] > 0 else None
    dominant = max(stages, key=lambda n: stages[n]["ms_per_step"]) if stages else None

    # ---- e2e through the public C ABI with pinned host buffers
    hbuf_in = b200.fn["host_alloc"](px * views * ring)
    hbuf_out = b200.fn["host_alloc"](px * 4 * 5)
    hin = np.ctypeslib.as_array(C.cast(hbuf_in, C.POINTER(C.c_uint8)), shape=(ring, px * views))
    frames_np = np.stack([f.image.reshape(-1) for f in frames])
    host_views = []
    for s in range(ring):
        arr = (_abi.View_c * views)()
        for k in range(views):
            f = frames[s + k]
            hin[s, k * px:(k + 1) * px] = frames_np[s + k]
            arr[k].image = hbuf_in + s * px * views + k * px
            arr[k].intrinsics = f.intrinsics.to_c()
            arr[k].pose = f.pose.to_c()
        host_views.append(arr)
    o_depth, o_norm, o_conf = hbuf_out, hbuf_out + 4 * px, hbuf_out + 16 * px

    def e2e_step(i):
        rc = b200.fn["estimate_bundle"](b200.ctx, host_views[i % ring], views, C.byref(ccfg),
                                        o_depth, o_norm, o_conf)
        if rc != 0:
            b200._check(rc)

    for i in range(args.warmup):
        e2e_step(i)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_maps = world * args.steps / e2e_s
    b200.fn["host_free"](hbuf_in)
    b200.fn["host_free"](hbuf_out)

    result = {
        "metric": METRIC, "value": round(maps_per_s, 3), "unit": "maps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u16",
        "data": "synthetic (device renderer of render.cpp value-noise plane, seed 1)",
        "config": {"workload": desc, "bundles_in_ring": ring,
                   "l2": "flushed before every timed step (256 MiB memset outside the events)",
                   "parallelism": f"bundle-parallel x{world} (no collective)"},
        "mde_per_s": round(maps_per_s * entries / 1e6, 1),
        "entries_per_bundle": entries, "levels": stats,
        "gpu_launches": int(launches_per_step * args.steps),
        "e2e": {"value": round(e2e_maps, 3), "unit": "maps/s", "h2d_bytes_per_step": px * views,
                "d2h_bytes_per_step": px * 20},
        "clocks": clocks.summary(),
        "stages": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                   for k, v in stages.items()},
    }
    if dominant is not None:
        st = stages[dominant]
        ach = st["gbs"] or 0.0
        result["roofline"] = {"kernel": dominant, "bound": "hbm", "achieved": round(ach, 1),
                              "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                              "traffic": None, "peak_source": peak_src,
                              "note": "achieved = algorithmic bytes / CUDA-event stage time; the "
                                      "sweep is FP64-issue-bound, see DESIGN.md"}
    return result


def cpu_reference(args, scene, cfgkw, steps, warmup):
    """The reference CPU implementation (oracle/_ref, the unmodified sources)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    import paper_2112_00821_b200 as pkg
    oracle = ref.load()
    cfg = make_config(pkg, **cfgkw)
    views = scene.get("views", 5)
    bundle, _, _ = oracle.render_plane_scene(
        scene["kind"], scene["width"], scene["height"], scene["focal"], scene["depth"], views,
        scene["step"], seed=1, tilt_deg=scene["tilt"], texture_scale=scene["texture"])
    for _ in range(warmup):
        oracle.estimate_bundle(bundle, cfg)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.estimate_bundle(bundle, cfg)
        times.append(time.perf_counter() - t0)
    cores = int(oracle.fn["worker_count"]())
    return steps / sum(times), cores, times


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--ring", type=int, default=8, help="distinct bundles cycled through")
    ap.add_argument("--cpu-baseline-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    scene, cfgkw, desc = WORKLOADS[args.workload]

    if args.impl == "reference":
        if rank != 0:
            return
        value, cores, times = cpu_reference(args, scene, cfgkw, args.steps, args.warmup)
        sample = f"{args.steps} full {args.workload.upper()} bundles, estimate_bundle only"
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "maps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 * sum(times) / len(times), 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+u16",
            "data": "synthetic (reference render_scene, seed 1)", "config": {"workload": desc},
            "cpu_baseline": {"value": round(value, 5), "unit": "maps/s", "cores": cores,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": round(value, 5), "unit": "maps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    result = run_b200(args, rank, world, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, times = cpu_reference(args, scene, cfgkw, args.cpu_baseline_steps, 0)
            result["cpu_baseline"] = {"value": round(v, 5), "unit": "maps/s", "cores": cores,
                                      "kind": "reference",
                                      "sample": f"{args.cpu_baseline_steps} {args.workload.upper()} "
                                                f"bundle(s) on {cores} host threads (oracle/_ref)"}
        except Exception as e:  # reported, never silently replaced
            result["cpu_baseline"] = {"value": None, "error": str(e)}
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


if __name__ == "__main__":
    main()
