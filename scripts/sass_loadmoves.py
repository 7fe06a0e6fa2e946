"""Flags global loads whose destination is consumed by a register MOV soon
after (the MOV stalls until the load returns): usage sass_loadmoves.py f.sass"""
import re, sys
ins = []
for ln in open(sys.argv[1]):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
    if m:
        ins.append((m.group(1), m.group(2).strip()))
bad = 0
for i, (addr, t) in enumerate(ins):
    m = re.search(r"\bLDG\S*\s+(R\d+)", t)
    if not m:
        continue
    r = m.group(1)
    for j in range(i + 1, min(i + 40, len(ins))):
        t2 = ins[j][1]
        if re.search(rf"\b{r}\b", t2.split(",", 1)[1] if "," in t2 else ""):
            if "MOV" in t2.split()[0] or (len(t2.split()) > 1 and "MOV" in t2.split()[1]):
                bad += 1
                print(addr, t, "->", ins[j][0], t2)
            break
print("load->move pairs:", bad)
