"""Summarise ncu evidence for profiles/: (1) the launch list of a bench run
(gpu__time_duration per launch, cold/serialised) -> per-kernel share; (2) one
`--set full` capture per kernel -> key metrics incl. DRAM traffic per launch.

usage: python scripts/ncu_summary.py <gpurun_out/ncu_WL dir> <out prefix> [command]
writes <prefix>_launches.txt and <prefix>_full.json
"""
import collections
import csv
import glob
import json
import os
import re
import subprocess
import sys

src, prefix = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else \
    "python bench.py --steps 2 --warmup 1 --inflight 1 --ring 2 --no-cpu-baseline"

rows = [r for r in csv.reader(open(os.path.join(src, "launches.csv"))) if len(r) > 10]
hdr = rows[0]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("fmvs::", "")
    name = name.replace("<unnamed>::", "").replace("unnamed>::", "")
    key = f"{name} grid{d['Grid Size']}"
    tot[key] += float(d["Metric Value"]) / 1e3
    cnt[key] += 1
all_us = sum(tot.values())
with open(prefix + "_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none launch list of\n"
            f"# `{cmd}`\n"
            "# (cold, serialised launches: compare shares, not absolute step time)\n"
            f"# {len(rows) - 1} launches, {all_us:.0f} us total\n")
    f.write(f"{'share':>6} {'total_us':>10} {'n':>5} {'avg_us':>9}  kernel\n")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{100 * v / all_us:5.1f}% {v:10.1f} {cnt[k]:5d} {v / cnt[k]:9.1f}  {k}\n")

keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for rep in sorted(glob.glob(os.path.join(src, "full_*.ncu-rep"))):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        m = {}
        for k in keys:
            if k in d:
                try:
                    m[k] = float(d[k].replace(",", ""))
                except ValueError:
                    m[k] = d[k]
                m[k + ".unit"] = u.get(k, "")
        tb = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tb += m.get(k, 0.0) * scale.get(m.get(k + ".unit", "byte"), 1)
        m["dram_bytes_per_launch"] = tb
        key = os.path.basename(rep).replace(".ncu-rep", "")
        key = key[len("full_"):] if key.startswith("full_") else key  # stage name (bench.py)
        out[key] = {"kernel": d["Kernel Name"],
                                                               "grid": d.get("launch__grid_size"), **m}
with open(prefix + "_full.json", "w") as f:
    json.dump(out, f, indent=1)
print(open(prefix + "_launches.txt").read()[:3500])
print(json.dumps({k: {kk: v.get(kk) for kk in ("kernel", "dram_bytes_per_launch", "gpu__time_duration.sum")}
                  for k, v in out.items()}, indent=1))
