export PYTHONPATH=$PWD
# round-1 K1 evidence: bench line (C4), launch list of the same command, one full ncu capture of the box kernel
python bench.py --config c4 > gpurun_out/b_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/k1_launches_c4.csv python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-fp64-peak > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"p1_box" -c 1 \
  -o gpurun_out/k1_box_full python tools/k1_ab.py cube6 8 0 > /dev/null 2>&1
tail -c 400 gpurun_out/b_c4.log
