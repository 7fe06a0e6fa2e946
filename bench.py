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

value : maps/s of the whole job: K bundles with inputs resident in HBM,
        `--inflight` contexts (one CUDA stream each) processing bundles round
        robin, device-timed with CUDA events (fork/join on a master stream);
        inputs larger than L2 (a ring of 16 distinct bundles); max over ranks.
latency_ms : one bundle alone, L2 flushed (256 MiB memset) before each step.
e2e   : the same metric through the public blocking C ABI
        (fmvs_estimate_bundle) from `--inflight` host threads with pinned HOST
        buffers: 5 images H2D + depth/normals/confidence D2H inside the timed
        region (wall clock around the calls).
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
    "c3": (dict(kind="slanted", width=1920, height=1080, focal=1920.0, depth=10.0, tilt=45.0,
                step=0.59, texture=0.1),
           dict(d_min=4.0, d_max=40.0, levels=1, max_planes=256, cost="ncc5", variant="plane", paths=8),
           "C3: slanted_scene 1920x1080 tilt 45deg, 5 views, 1 level, 256 planes (dense), NCC 5x5, "
           "SGM pi 8 paths, confidence"),
    # C5: the C2 scene as a stream of 512 max-overlap bundles from a 516-frame
    # lateral track, sharded contiguously over ranks (strong scaling)
    "c5": (dict(kind="slanted", width=1920, height=1080, focal=1920.0, depth=10.0, tilt=30.0,
                step=0.59, texture=0.1, stream_frames=516),
           dict(d_min=4.0, d_max=40.0, levels=3, max_planes=128, cost="census5", variant="sn", paths=8),
           "C5: stream of 512 C2 bundles (516-frame lateral track, max overlap), sharded over GPUs"),
    # C2 scene with the other SGM variants / the NCC matcher (variant coverage)
    "c2pg": (dict(kind="slanted", width=1920, height=1080, focal=1920.0, depth=10.0, tilt=30.0,
                  step=0.59, texture=0.1),
             dict(d_min=4.0, d_max=40.0, levels=3, max_planes=128, cost="census5", variant="pg", paths=8),
             "C2 with SGM pi-pg (path gradient) 8 paths"),
    "c2ncc": (dict(kind="slanted", width=1920, height=1080, focal=1920.0, depth=10.0, tilt=30.0,
                   step=0.59, texture=0.1),
              dict(d_min=4.0, d_max=40.0, levels=3, max_planes=128, cost="ncc5", variant="sn", paths=8),
              "C2 with the NCC 5x5 matcher, SGM pi-sn 8 paths"),
    "c4": (dict(kind="slanted", width=3840, height=2160, focal=3840.0, depth=10.0, tilt=30.0,
                step=0.59, texture=0.05),
           dict(d_min=4.0, d_max=40.0, levels=3, max_planes=192, cost="ncc5", variant="plane", paths=8),
           "C4: slanted_scene 3840x2160 f=3840 tilt 30deg, 5 views, 3 levels, max_planes 192, "
           "NCC 5x5, SGM pi 8 paths"),
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
    """nvidia-smi clocks / throttle reasons, sampled every 100 ms from before
    the warm-up on; summary() keeps only the samples that fall inside the
    marked timed regions (the device-timed region and the e2e region)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (host time, fields)
        self.regions = []
        self.proc = None

    def start(self):
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
                self.samples.append((time.time(), parts))

    def region(self, t0, t1):
        self.regions.append((t0, t1))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        inside = [p for t, p in self.samples if any(a <= t <= b for a, b in self.regions)]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in inside if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside)}


def render_frames(b200, scene, frames):
    """Renders a lateral track of `frames` views on the device (render.cpp)."""
    bundle, _, _ = b200.render_plane_scene(
        scene["kind"], scene["width"], scene["height"], scene["focal"], scene["depth"], frames,
        scene["step"], seed=1, tilt_deg=scene["tilt"], texture_scale=scene["texture"])
    return bundle


def alg_bytes(stage, stats, n_views, paths, sn=False):
    """Algorithmic HBM bytes of one stage per bundle, summed over the levels
    it runs on: every map read or written once, cost
    volumes at the reference's widths (u16 cost, u32 aggregate), 8 B of
    ragged-layout metadata per pixel. stats[0] is level 0 (finest)."""
    L = len(stats)
    px = [lv["width"] * lv["height"] for lv in stats]
    ent = [lv["entries"] for lv in stats]
    tail = range(L) if sn else [0]   # levels that compute normals (SN needs them as priors)
    if stage == "sweep_l0":
        return ent[0] * 2 + px[0] * (8 + n_views)   # u16 cost per hypothesis
    if stage == "sweep":
        return sum(ent[l] * 2 + px[l] * (8 + n_views) for l in range(1, L))
    if stage == "zero":         # the u32 SGM accumulator of every level, zeroed
        return sum(ent[l] * 4 for l in range(L))
    if stage == "sgm_l0":
        return ent[0] * (2 * paths + 4) + px[0] * paths * 9
    if stage == "sgm":
        return sum(ent[l] * (2 * paths + 4) + px[l] * paths * 9 for l in range(1, L))
    if stage == "pyramid":      # blur + ceil-halve: read level l-1, write level l, every view
        return sum(n_views * (px[l - 1] + px[l]) for l in range(1, L))
    if stage == "quads":        # matching views: 1 B in, 4 B packed bilinear taps out
        return sum((n_views - 1) * px[l] * 5 for l in range(L))
    if stage == "range":        # prior depth (coarser level) in; meta + row totals out
        return sum(px[l] * 8 + (4 * px[l + 1] if l + 1 < L else 0) for l in range(L))
    if stage == "offsets":      # SN: prior depth + normals (coarser) in, 4 x int16 out
        return sum(16 * px[l + 1] + 8 * px[l] for l in range(L - 1)) if sn else 0
    if stage == "wta":          # aggregate + meta in, depth out
        return sum(ent[l] * 4 + px[l] * (8 + 4) for l in range(L))
    if stage == "median":
        return sum(px[l] * 8 for l in range(L))
    if stage == "normals":      # depth in, raw normals out
        return sum(px[l] * 16 for l in tail)
    if stage == "smooth_conf":  # raw normals + image in, normals out (+ confidence at level 0)
        return sum(px[l] * (12 + 1 + 12) + (4 * px[l] if l == 0 else 0) for l in tail)
    return 0


# ncu --set full captures of the bench command, one per (workload, stage)
# (scripts/ncu_capture.sh -> scripts/ncu_summary.py): DRAM bytes of one launch
# of the stage's kernel and its SM-side utilisation. Read from the committed
# summary of THIS workload only; never measured under ncu here, never
# borrowed from another workload or kernel (null when no capture exists).
NCU_DIR = os.path.join(ROOT, "profiles", "r2")


def ncu_capture(workload, stage):
    path = os.path.join(NCU_DIR, f"ncu_{workload}_full.json")
    try:
        with open(path) as f:
            m = json.load(f)[stage]
    except (OSError, KeyError, ValueError):
        return None, None
    return m, os.path.relpath(path, ROOT)


def roofline_entry(stage, st, peak, peak_src, workload):
    ach = st["gbs"] or 0.0
    e = {"kernel": stage, "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
         "frac": round(ach / peak, 4), "traffic": None, "peak_source": peak_src,
         "alg_bytes_per_launch": st["alg_bytes"], "avg_launch_ms": st["ms_per_step"]}
    m, src = ncu_capture(workload, stage)
    if m is not None:
        e["traffic"] = int(m["dram_bytes_per_launch"])
        e["traffic_source"] = (f"{src}: dram__bytes_read.sum + dram__bytes_write.sum of one "
                               f"ncu --set full launch of {m['kernel'].split('(')[0]} ({workload})")
        e["sm_throughput_pct"] = m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed")
        # the binding resource of the sweeps is instruction issue, not HBM
        # (SURVEY §8d / BASELINE.md §3): its fraction from the same capture
        e["compute_roofline"] = {
            "resource": "SM issue slots (warp-instructions / cycle / SMSP)",
            "frac": round(float(m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0)) / 100, 4),
            "fp64_pipe_frac": round(float(m.get(
                "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 0.0)) / 100, 4),
            "alu_pipe_frac": round(float(m.get(
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 0.0)) / 100, 4),
            "warps_active_frac": round(float(m.get(
                "sm__warps_active.avg.pct_of_peak_sustained_active", 0.0)) / 100, 4),
            "source": f"ncu --set full capture ({src})"}
    if stage.startswith("sweep"):
        e["note"] = ("achieved = algorithmic bytes (2 B cost per hypothesis + 8 B meta + 1 B per view "
                     "per pixel) / CUDA-event launch time; the sweep is "
                     "ALU-issue-bound (certified FP32/integer matching + FP64 tie fallback), not "
                     "HBM-bound: see DESIGN.md section 5")
    else:
        e["note"] = ("achieved = algorithmic bytes (per hypothesis and path 2 B cost + 4 B "
                     "aggregate, per pixel and path 9 B) / CUDA-event launch time")
    return e


def output_digest(depth, normals, confidence) -> str:
    """sha256 over the raw bytes of one bundle's depth, normals and confidence
    maps (row-major float32, normals xyz-interleaved)."""
    import hashlib
    h = hashlib.sha256()
    for a in (depth, normals, confidence):
        h.update(np.ascontiguousarray(a, dtype=np.float32).tobytes())
    return h.hexdigest()


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous shard of a bundle stream for one rank (no collective needed:
    bundles are independent)."""
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


# Test hook: FMVS_BENCH_SHARE_DEVICE=1 runs every rank on cuda:0 with the gloo
# backend, so the N>1 code path (sharding, barriers, max-over-ranks) can be
# exercised on a single-GPU box. Never used for reported numbers.
SHARE_DEVICE = os.environ.get("FMVS_BENCH_SHARE_DEVICE") == "1"


def reduce_max(value: float, world: int, device: str = "cpu") -> float:
    """Max over ranks of a per-rank time (the timing rule); plumbing only."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    if SHARE_DEVICE:
        device = "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_b200(args, rank, world, device):
    import threading as th
    import torch
    import paper_2112_00821_b200 as pkg
    from paper_2112_00821_b200 import Backend, _abi

    scene, cfgkw, desc = WORKLOADS[args.workload]
    views = scene.get("views", 5)
    dev = f"cuda:{device}"
    torch.cuda.set_device(device)
    libpath = os.environ.get("FMVS_LIB") or os.path.join(ROOT, "paper_2112_00821_b200", "_lib", "libfmvs.so")
    if not os.path.exists(libpath):
        raise RuntimeError("libfmvs.so not built (run __graft_entry__.build())")
    M = max(1, args.inflight)
    ctxs = [Backend(libpath, "fmvs_", device) for _ in range(M)]
    b200 = ctxs[0]
    cfg = make_config(pkg, **cfgkw)
    ccfg = cfg.to_c()
    stream = scene.get("stream_frames")
    if stream:
        # C5: this rank's contiguous shard of the 512-bundle stream
        mine = shard(stream - views + 1, rank, world)
        track = render_frames(b200, scene, stream)
        frames = track[mine.start:mine.stop + views - 1]
        ring = len(mine)
        n_steps, job_bundles = ring, stream - views + 1
    else:
        ring = args.ring
        frames = render_frames(b200, scene, ring + views - 1)
        n_steps, job_bundles = args.steps, world * args.steps
    h, w = frames[0].image.shape
    px = w * h
    d_frames = torch.from_numpy(np.stack([f.image for f in frames])).to(dev)
    outs = [(torch.empty((h, w), dtype=torch.float32, device=dev),
             torch.empty((h, w, 3), dtype=torch.float32, device=dev),
             torch.empty((h, w), dtype=torch.float32, device=dev)) for _ in range(M)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    streams = [torch.cuda.ExternalStream(c.fn["ctx_stream"](c.ctx), device=dev) for c in ctxs]

    def dev_views(i):
        s0 = i % ring
        arr = (_abi.View_c * views)()
        for k in range(views):
            f = frames[s0 + k]
            arr[k].image = d_frames[s0 + k].data_ptr()
            arr[k].intrinsics = f.intrinsics.to_c()
            arr[k].pose = f.pose.to_c()
        return arr

    vlist = [dev_views(i) for i in range(ring)]

    def step(ci, i):
        c = ctxs[ci]
        o = outs[ci]
        rc = c.fn["estimate_bundle_device"](c.ctx, vlist[i % ring], views, C.byref(ccfg),
                                            o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr())
        if rc != 0:
            c._check(rc)

    def sync_all():
        for c in ctxs:
            c._check(c.fn["ctx_synchronize"](c.ctx))

    clocks = ClockSampler(device).start()
    # warmup (every context, every ring slot touched once)
    for i in range(max(args.warmup, 1) * M):
        step(i % M, i)
    sync_all()
    stats = b200.level_stats()
    launches_per_step = b200.last_launch_count()
    entries = sum(lv["entries"] for lv in stats)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(device)

    def max_over_ranks(v):
        return reduce_max(v, world, dev)

    # ---- value: K bundles, M contexts in flight (round robin), device-timed
    master = torch.cuda.Stream(device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event() for _ in range(M)]
    barrier()
    t_region = time.time()
    ev0.record(master)
    for st in streams:
        st.wait_event(ev0)
    for i in range(n_steps):
        step(i % M, args.warmup * M + i)
    for e, st in zip(ends, streams):
        e.record(st)
        master.wait_event(e)
    ev1.record(master)
    ev1.synchronize()
    clocks.region(t_region, time.time())
    # digest of the last timed bundle's outputs (tests/test_fullsize_gpu.py
    # recomputes it with the oracle on the same frames)
    last = n_steps - 1
    digest = {"bundle": (args.warmup * M + last) % ring,
              "sha256": output_digest(*(t.cpu().numpy() for t in outs[last % M]))}
    total_ms = max_over_ranks(ev0.elapsed_time(ev1))
    maps_per_s = job_bundles * 1000.0 / total_ms

    # ---- latency: one bundle at a time, L2 flushed before every timed step
    lat = []
    s0 = streams[0]
    for i in range(min(args.steps, 10)):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s0):
            flush.zero_()
            a_.record(s0)
        step(0, i)
        with torch.cuda.stream(s0):
            b_.record(s0)
        b_.synchronize()
        lat.append(a_.elapsed_time(b_))

    # ---- per-stage CUDA-event timing pass (roofline of the dominant kernel)
    b200.fn["ctx_set_timing"](b200.ctx, 1)
    b200.fn["ctx_stage_reset"](b200.ctx)
    nprof = 5
    for i in range(nprof):
        with torch.cuda.stream(s0):
            flush.zero_()
        step(0, i)
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
        b = alg_bytes(name, stats, views, cfg.sgm.paths, sn=cfg.sgm.variant == pkg.SgmVariant.SurfaceNormal)
        st["alg_bytes"] = b
        st["gbs"] = b / (st["ms_per_step"] * 1e6) if b and st["ms_per_step"] > 0 else None
    dominant = max(stages, key=lambda n: stages[n]["ms_per_step"]) if stages else None

    # ---- e2e: the public blocking C ABI (fmvs_estimate_bundle) from M host
    # threads, pinned HOST inputs/outputs, H2D + D2H inside the timed region
    hin = b200.fn["host_alloc"](px * views * ring)
    hout = [b200.fn["host_alloc"](px * 20) for _ in range(M)]
    hin_np = np.ctypeslib.as_array(C.cast(hin, C.POINTER(C.c_uint8)), shape=(ring, px * views))
    host_views = []
    for s_ in range(ring):
        arr = (_abi.View_c * views)()
        for k in range(views):
            f = frames[s_ + k]
            hin_np[s_, k * px:(k + 1) * px] = f.image.reshape(-1)
            arr[k].image = hin + s_ * px * views + k * px
            arr[k].intrinsics = f.intrinsics.to_c()
            arr[k].pose = f.pose.to_c()
        host_views.append(arr)

    def e2e_worker(ci, n, first_i, errs):
        c = ctxs[ci]
        o = hout[ci]
        try:
            for j in range(n):
                rc = c.fn["estimate_bundle"](c.ctx, host_views[(first_i + j * M) % ring], views,
                                             C.byref(ccfg), o, o + 4 * px, o + 16 * px)
                if rc != 0:
                    c._check(rc)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    def run_e2e(nsteps):
        errs = []
        per = [nsteps // M + (1 if ci < nsteps % M else 0) for ci in range(M)]
        ts = [th.Thread(target=e2e_worker, args=(ci, per[ci], ci, errs)) for ci in range(M)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        return time.perf_counter() - t0

    run_e2e(max(args.warmup, 1) * M)
    barrier()
    t_region = time.time()
    e2e_s = max_over_ranks(run_e2e(n_steps))
    clocks.region(t_region, time.time())
    clocks.stop()
    e2e_maps = job_bundles / e2e_s
    b200.fn["host_free"](hin)
    for o in hout:
        b200.fn["host_free"](o)

    result = {
        "metric": METRIC, "value": round(maps_per_s, 3), "unit": "maps/s", "n_gpus": world,
        "steps": n_steps, "warmup": args.warmup, "ms_per_step": round(total_ms / n_steps, 4),
        "higher_is_better": True, "scaling": "strong" if stream else "weak", "vs_baseline": None,
        "dtype": "f64+u16",
        "data": "synthetic (device renderer of render.cpp value-noise plane, seed 1)",
        "config": {"workload": desc, "bundles_in_flight": M, "bundles_in_ring": ring,
                   "l2": (f"inputs larger than L2: ring of {ring} distinct bundles "
                          f"({ring * views * px / 1e6:.0f} MB of frames), per-bundle working set "
                          f"> L2; latency_ms is measured with a 256 MiB L2 flush before each step"),
                   "parallelism": f"bundle-parallel x{world} GPUs x {M} streams (no collective)"},
        "mde_per_s": round(maps_per_s * entries / 1e6, 1),
        "entries_per_bundle": entries, "levels": stats,
        "latency_ms": round(statistics.median(lat), 3),
        "output_digest": digest,
        "gpu_launches": int(launches_per_step * args.steps),
        "e2e": {"value": round(e2e_maps, 3), "unit": "maps/s", "h2d_bytes_per_step": px * views,
                "d2h_bytes_per_step": px * 20, "host_threads": M},
        "clocks": clocks.summary(),
        "stages": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                   for k, v in stages.items()},
    }
    if dominant is not None:
        result["roofline"] = roofline_entry(dominant, stages[dominant], peak, peak_src, args.workload)
        if "sgm_l0" in stages and dominant != "sgm_l0":
            # the north star names both the sweep and SGM; SGM is the HBM/L2-facing one
            result["roofline_sgm"] = roofline_entry("sgm_l0", stages["sgm_l0"], peak, peak_src,
                                                    args.workload)
    for c in ctxs:
        c.close()
    return result


def cpu_reference(args, scene, cfgkw, steps, warmup, threads=None):
    """The reference CPU implementation (oracle/_ref, the unmodified sources),
    on `threads` workers (FASSMVS_THREADS, parallel.cpp:10-18; default: every
    host thread)."""
    if threads:
        os.environ["FASSMVS_THREADS"] = str(threads)
    else:
        os.environ.pop("FASSMVS_THREADS", None)
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


def self_spawn(n: int) -> int:
    """Re-launches this command under torch.distributed.run with one rank per
    GPU (the driver's own launch form); fails loudly when fewer than n GPUs
    are visible (never a silent 1-GPU run)."""
    import socket
    if not SHARE_DEVICE:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} requested but {have} GPU(s) visible", file=sys.stderr)
            return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--ring", type=int, default=16, help="distinct bundles cycled through")
    ap.add_argument("--inflight", type=int, default=5, help="bundles in flight (contexts/streams; also the e2e host threads)")
    ap.add_argument("--cpu-baseline-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-1t", action="store_true",
                    help="also time one bundle of the reference on ONE host thread (~1 min at C2)")
    ap.add_argument("--cpu-threads", type=int, default=0,
                    help="reference arm: host threads (default: all)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: one process per GPU, launched here
        sys.exit(self_spawn(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    scene, cfgkw, desc = WORKLOADS[args.workload]

    if args.impl == "reference":
        if rank != 0:
            return
        value, cores, times = cpu_reference(args, scene, cfgkw, args.steps, args.warmup,
                                            args.cpu_threads or None)
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
        if SHARE_DEVICE:
            local = 0
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    result = run_b200(args, rank, world, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, times = cpu_reference(args, scene, cfgkw, args.cpu_baseline_steps, 0)
            result["cpu_baseline"] = {"value": round(v, 5), "unit": "maps/s", "cores": cores,
                                      "kind": "reference", "host_threads": os.cpu_count(),
                                      "sample": f"{args.cpu_baseline_steps} {args.workload.upper()} "
                                                f"bundle(s) on {cores} host threads (oracle/_ref)"}
            if args.cpu_baseline_1t:
                v1, c1, _ = cpu_reference(args, scene, cfgkw, 1, 0, threads=1)
                result["cpu_baseline"]["single_thread"] = {
                    "value": round(v1, 5), "unit": "maps/s", "cores": c1,
                    "sample": f"1 {args.workload.upper()} bundle on 1 host thread (FASSMVS_THREADS=1)"}
        except Exception as e:  # reported, never silently replaced
            result["cpu_baseline"] = {"value": None, "error": str(e)}
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


if __name__ == "__main__":
    main()
