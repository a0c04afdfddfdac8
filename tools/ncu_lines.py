"""Per-source-line stall samples and executed instructions of an ncu report
(source page, cuda+sass). usage: python tools/ncu_lines.py REPORT [min_pct]"""
import csv, subprocess, sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
iw = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
it = hdr.index("Avg. Threads Executed") if "Avg. Threads Executed" in hdr else None
def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


lines = [r for r in rows[rows.index(hdr) + 1:] if r and r[0] not in ("", "Line No") and r[0].isdigit()]
tw = sum(num(r[iw]) for r in lines) or 1
te = sum(num(r[ie]) for r in lines) or 1
print(f"total warp-instructions {te:.0f}, stall samples {tw:.0f}")
for r in lines:
    w, e = num(r[iw]), num(r[ie])
    if 100 * w / tw >= thr or 100 * e / te >= thr:
        th = r[it] if it is not None else ""
        print(f"{r[0]:>5} stall {100 * w / tw:5.1f}%  inst {100 * e / te:5.1f}%  thr {th:>6}  {r[1].strip()[:90]}")
