export PYTHONPATH=$PWD
# K1 default (variant 0 = box kernel) vs the round-1 walk (9) and tuning builds (tools/build_variant.sh)
timeout 120 python tools/k1_ab.py cube6 8 0 9 2>&1 | grep variant
for v in "$@"; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 120 python tools/k1_ab.py cube6 8 0 2>&1 | tail -1 | sed "s/^/$v /"; done
timeout 120 python tools/k1_ab.py cubes2 7 0 9 2>&1 | tail -2
timeout 120 python tools/k1_ab.py single-tet 9 0 9 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" 2>&1 | tail -2
