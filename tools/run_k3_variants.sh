#!/bin/bash
# K3 A/B on the GPU box: bitwise hash + C5 kernel time of the default build,
# the per-cube kernel (--variant 1) and variant builds
# (tools/build_variant.sh NAME k_n1_fold.cu "-D...").
#   bash tools/run_k3_variants.sh NAME1 NAME2 ...
export PYTHONPATH=$PWD
V=paper_2404_08371_b200/_lib/variants
python tools/k3_hash.py
for v in "$@"; do TETMF_LIB=$V/libtetmf_$v.so python tools/k3_hash.py; done
run() { python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-subrecords $2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', round(d['value'],2), 'GDoF/s kernel', round(r['kernel_ms'],3), 'ms frac', round(r['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
  run default ""
  run cubes "--variant 1"
  for v in "$@"; do TETMF_LIB=$V/libtetmf_$v.so run $v ""; done
done
