export PYTHONPATH=$PWD
mkdir -p gpurun_out
for c in 32 40 48 64 96 128 32; do
  TETMF_N1F2_CHUNK_STEPS=$c python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-subrecords --no-fp64-peak 2>/dev/null | tail -1 > gpurun_out/k3c5_chunk_$c.json
  python - <<P
import json
d=json.load(open("gpurun_out/k3c5_chunk_$c.json"))
print("chunk $c", d["value"], d["ms_per_step"], d["roofline"].get("kernel_ms"), d["clocks"]["sm_mhz"], flush=True)
P
done | tee gpurun_out/k3c5_chunk_sweep.txt
