"""Sum ncu source-page instruction counts / stall samples over line ranges.
usage: ncu_ranges.py rep file.cu name:a-b [name:a-b ...]"""
import csv, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for r in sys.argv[3:]:
    n, ab = r.split(":"); a, b = ab.split("-"); ranges.append((n, int(a), int(b)))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
file = None; hdr = None; tot_i = 0; tot_s = 0; acc = {n: [0, 0] for n, _, _ in ranges}; other = {}
for row in csv.reader(src.splitlines()):
    if not row: continue
    if row[0] == "File Path": file = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or row[0] == "": continue
    try: ln = int(row[0]); s = int(row[4]); i = int(row[7])
    except (ValueError, IndexError): continue
    tot_i += i; tot_s += s
    hit = False
    if file == fname:
        for n, a, b in ranges:
            if a <= ln <= b:
                acc[n][0] += i; acc[n][1] += s; hit = True; break
    if not hit:
        k = file if file != fname else f"{fname}:other"
        other.setdefault(k, [0, 0]); other[k][0] += i; other[k][1] += s
print(f"total warp instr {tot_i/1e6:.1f}M")
for n, (i, s) in list(acc.items()) + sorted(other.items(), key=lambda kv: -kv[1][0]):
    print(f"{n:28s} {100*i/tot_i:5.1f}% inst {i/1e6:8.1f}M  {100*s/max(tot_s,1):5.1f}% stall")
