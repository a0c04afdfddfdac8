"""Per-kernel launch counts and mean ncu durations of a
`ncu --metrics gpu__time_duration.sum --csv` log: python tools/launch_table.py FILE"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
c, t = collections.OrderedDict(), collections.defaultdict(float)
for r in rows:
    k = r[4].split("(")[0].replace("(anonymous namespace)::", "")
    c[k] = c.get(k, 0) + 1
    t[k] += float(r[-1])
for k, v in c.items():
    print(f"  {v:3d}  {k:50s} {t[k] / v / 1000:8.2f} us/launch (ncu, serialised)")
