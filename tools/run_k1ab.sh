#!/bin/bash
# A/B sweep of K1 stream-kernel builds (tools/build_variant.sh k1*) on the GPU box
export PYTHONPATH=.
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so
  echo "== $v"
  TETMF_LIB=$lib timeout 60 python tools/k1_ab.py cube6 8 0 3
  TETMF_LIB=$lib timeout 60 python tools/k1_ab.py cubes2 7 0 3
done
