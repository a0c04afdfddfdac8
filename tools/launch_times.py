"""Per-launch kernel durations from an ncu --csv launch list (gpu__time_duration.sum).
usage: python tools/launch_times.py FILE.csv [name-substring]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i]
kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
sub = sys.argv[2] if len(sys.argv) > 2 else ""
tot = 0.0
for r in rows[i + 1:]:
    if len(r) == len(hdr) and r[mn] == "gpu__time_duration.sum" and sub in r[kn]:
        v = float(r[mv].replace(",", ""))
        tot += v
        print(f"{r[kn][:60]:60s} {v:12.1f}")
print("total", tot)
