"""Per-opcode warp-stall breakdown from an ncu report's source page.
usage: python tools/ncu_stalls.py REPORT.ncu-rep"""
import csv, subprocess, sys
from collections import Counter
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia = hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons}
data = []
for r in rows[2:]:
    if r and r[0].startswith("Kernel"):
        break  # first kernel only
    if len(r) == len(hdr) and r[0] != "Address":
        data.append(r)
c = {}
for r in data:
    s = r[ia].strip()
    op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
    cc = c.setdefault(op, Counter())
    for h in reasons:
        cc[h] += int(r[idx[h]] or 0)
allr = Counter()
for v in c.values():
    allr += v
tot = sum(allr.values()) or 1
print("overall", [(k[6:], round(100 * v / tot, 1)) for k, v in allr.most_common(9)])
for op, v in sorted(c.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
    t = sum(v.values())
    print(f"{op:10s} {100 * t / tot:5.1f}%", [(k[6:], round(100 * x / tot, 1)) for k, x in v.most_common(4)])
