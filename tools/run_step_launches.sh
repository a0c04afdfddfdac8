export PYTHONPATH=$PWD
# per-launch durations (ncu launch list) of one apply: mesh level form-variant
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/k1_ab.py ${1:-cube6} ${2:-8} 0 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>14 and r[0].isdigit()]
for r in rows[-6:]: print(r[4][:60], r[-1])
"
