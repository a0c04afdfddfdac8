export PYTHONPATH=$PWD
timeout 120 python tools/k1_ab.py cube6 8 0 2>&1 | grep variant
for v in "$@"; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 120 python tools/k1_ab.py cube6 8 0 2>&1 | grep variant | sed "s/^/$v /"; done
for v in "$@"; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 120 python tools/k1_ab.py cubes2 7 0 2>&1 | grep variant | sed "s/^/$v /"; done
TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$1.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" 2>&1 | tail -1
