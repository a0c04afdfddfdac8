#!/bin/bash
# End-of-session evidence on one B200 (gpurun): GPU tests, smoke, the default
# bench line (config 5 + c4 / c2l / p2v sub-records), the reference arm, the
# launch list of one default bench step, and one ncu --set full capture of
# the K2 walk kernel at c2l.   bash tools/run_evidence.sh TAG
TAG=${1:-r2}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputests.log 2>&1; tail -1 gpurun_out/${TAG}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -3 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log > gpurun_out/${TAG}_bench_ref.json
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-subrecords > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c5.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-subrecords --no-fp64-peak > /dev/null 2>&1
python bench.py --config c2l --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c2l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:p1k_cube -s 3 -c 1 -o gpurun_out/${TAG}_k2cube \
    python bench.py --config c2l --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
