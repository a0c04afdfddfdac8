#!/bin/bash
# correctness repeat runs of K1 stream builds
export PYTHONPATH=.
for v in "$@"; do
  lib=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so
  echo "== $v"
  for mesh in "cube6 8" "single-tet 8" "cube6 7" "cubes2 6"; do
    TETMF_LIB=$lib timeout 60 python tools/k1_ab.py $mesh 0 3 3 | grep "variant 3"
  done
done
