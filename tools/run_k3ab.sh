#!/bin/bash
# A/B of K3 builds on C5 (bench.py kernel time), args: variant lib names
export PYTHONPATH=.
for v in "$@"; do
  lib=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so
  TETMF_LIB=$lib timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64-peak > gpurun_out/k3ab_$v.json 2> gpurun_out/k3ab_$v.err
  python tools/bline.py gpurun_out/k3ab_$v.json
done
