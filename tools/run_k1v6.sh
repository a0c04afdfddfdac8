export PYTHONPATH=$PWD
# K1 variant 6 A/B: default build and tuning builds (tools/build_variant.sh)
timeout 120 python tools/k1_ab.py cube6 8 0 7 8 2>&1 | tail -3
for v in "$@"; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 120 python tools/k1_ab.py cube6 8 0 8 2>&1 | tail -1 | sed "s/^/$v /"; done
timeout 120 python tools/k1_ab.py cubes2 7 0 7 8 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" 2>&1 | tail -2
