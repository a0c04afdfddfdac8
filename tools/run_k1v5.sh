export PYTHONPATH=$PWD
# K1 variant 5 A/B: default build and tuning builds (tools/build_variant.sh)
python tools/k1_ab.py cube6 8 0 5 2>&1 | tail -2
for v in "$@"; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so python tools/k1_ab.py cube6 8 0 5 2>&1 | tail -1 | sed "s/^/$v /"; done
python tools/k1_ab.py cubes2 7 0 5 2>&1 | tail -1
python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" 2>&1 | tail -2
# timeout 300 ncu --set full --clock-control none --import-source on -k regex:"p1_interior|p1_face" -c 2 \
#  -o gpurun_out/k1v5_full python tools/k1_ab.py cube6 8 5 > gpurun_out/k1v5_ncu.log 2>&1
