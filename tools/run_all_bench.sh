export PYTHONPATH=$PWD
# all bench lines of the round (each config once), the reference arm, c5 launch list
for c in c1 c2 c3 c4 p2v c5; do python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log > gpurun_out/bench_$c.json; done
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
for c in c1 c2 c3 c4 p2v c5 ref; do python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d.get('roofline') or {}
print('$c', round(d['value'],4), d.get('ms_per_step'), r.get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks'))"; done
