"""Print stall breakdown + top source lines of an ncu report (local analysis helper)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); h = r[0]; d = dict(zip(h, r[2]))
print(d["Kernel Name"], "grid", d["launch__grid_size"], "regs", d.get("launch__registers_per_thread"))
out = []
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
        try: out.append((float(d[k]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError: pass
print("stalls/issue:", ", ".join(f"{k} {v:.2f}" for v, k in sorted(out, reverse=True)[:8]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
          "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]:
    print(" ", k, d.get(k))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
stats = []; file = None; hdr = None
for row in csv.reader(src.splitlines()):
    if not row: continue
    if row[0] == "File Path": file = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or row[0] == "": continue
    try: s = int(row[4]); i = int(row[7])
    except (ValueError, IndexError): continue
    stats.append((s, i, f"{file}:{row[0]}", row[1].strip()[:80]))
ts = sum(x[0] for x in stats) or 1; ti = sum(x[1] for x in stats) or 1
print(f"warp instr {ti/1e6:.1f}M")
for x in sorted(stats, reverse=True)[:top]:
    print(f"{100*x[0]/ts:5.1f}% smp {100*x[1]/ti:5.1f}% inst  {x[2]:22s} {x[3]}")
