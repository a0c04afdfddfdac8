#!/bin/bash
# A/B of programmatic dependent launch (TETMF_PDL=0 / 1): back-to-back applies
# of the configurations whose apply is two short kernels (K1 / K2 + K4).
# bash tools/pdl_ab.sh  (one B200; writes gpurun_out/pdl_ab.txt)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for rep in 1 2; do for pdl in 0 1 2 3; do TETMF_PDL=$pdl python tools/pdl_ab.py 2>&1 | grep -v Warning; done; done | tee gpurun_out/pdl_ab.txt
