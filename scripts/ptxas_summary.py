"""Per-kernel registers / spills / smem from an nvcc -Xptxas -v log."""
import re, subprocess, sys
cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"fmvs::k::\(anonymous namespace\)::", "", cur)
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if len(sys.argv) < 3 or sys.argv[2] in cur:
            print(f"{m.group(1):>4} regs  {spill:22s} {cur[:110]}")
        cur = None
