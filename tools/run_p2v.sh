#!/bin/bash
# P2V builds: parity tests + timing, args: variant lib names ("" = default lib)
export PYTHONPATH=.
for v in "$@"; do
  echo "== $v"
  if [ -n "$v" ] && [ "$v" != "default" ]; then export TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so; else unset TETMF_LIB; fi
  timeout 300 python -m pytest tests/test_gpu_p2v.py -x -q 2>&1 | tail -1
  timeout 300 python tools/p2v_time.py
done
