export PYTHONPATH=$PWD
# end-of-session evidence: GPU tests, smoke, every bench line, reference arm, K1 / K3 ncu evidence
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_gputests.log 2>&1; tail -1 gpurun_out/final_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -3 gpurun_out/final_smoke.log
bash tools/run_all_bench.sh
bash tools/run_profiles_k1.sh > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/k3_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-fp64-peak > /dev/null 2>&1
echo done
