export PYTHONPATH=$PWD
V=paper_2404_08371_b200/_lib/variants
python tools/k2_ab.py --c2l-only 0 3 2>&1 | grep c2l
for v in "$@"; do echo "== $v"; TETMF_LIB=$V/libtetmf_$v.so python tools/k2_ab.py --c2l-only 0 2>&1 | grep c2l; done
