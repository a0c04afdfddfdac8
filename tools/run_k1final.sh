export PYTHONPATH=$PWD
# K1 head-to-head: repeated runs of the candidate builds / variants
for rep in 1 2 3; do
for mesh in "cube6 8" "cubes2 7" "single-tet 9"; do
  timeout 120 python tools/k1_ab.py $mesh 0 2>&1 | tail -1
  for v in c4 c6; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 120 python tools/k1_ab.py $mesh 5 2>&1 | tail -1 | sed "s/^/$v /"; done
  for v in sw2 sw2c128 sw2r6; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 120 python tools/k1_ab.py $mesh 6 2>&1 | tail -1 | sed "s/^/$v /"; done
done; done
