#!/bin/bash
# repeated correctness runs (cube6 L8) of K1 stream builds
export PYTHONPATH=.
for v in "$@"; do
  lib=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so
  echo "== $v"
  TETMF_LIB=$lib timeout 90 python tools/k1_ab.py cube6 8 0 3 3 3 3 3 3 3 3 | grep "variant 3" | awk '{print $NF}' | paste -sd' '
done
