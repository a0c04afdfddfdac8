#!/bin/bash
# K2 A/B on the GPU box: c2l (P1K cube6 L8) kernel time of the default build
# and of variant builds (tools/build_variant.sh NAME k_p1k_gather.cu "-D...").
export PYTHONPATH=$PWD
V=paper_2404_08371_b200/_lib/variants
run() { python bench.py --config c2l --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', round(d['value'],2), 'GDoF/s kernel', round(r['kernel_ms'],4), 'ms frac', round(r['frac'],4))"; }
run default
for v in "$@"; do TETMF_LIB=$V/libtetmf_$v.so run $v; done
