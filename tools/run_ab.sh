#!/bin/bash
# A/B of variant builds of one config on the GPU box:
#   bash tools/run_ab.sh CONFIG NAME1 NAME2 ...   (tools/build_variant.sh NAME SOURCE.cu "-D...")
export PYTHONPATH=$PWD
V=paper_2404_08371_b200/_lib/variants
C=$1; shift
run() { python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', round(d['value'],2), 'GDoF/s kernel', round(r['kernel_ms'],4), 'ms frac', round(r['frac'],4), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  run default
  for v in "$@"; do TETMF_LIB=$V/libtetmf_$v.so run $v; done
done
