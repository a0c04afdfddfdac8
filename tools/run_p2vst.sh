export PYTHONPATH=$PWD
python tools/p2v_time.py 2>&1 | tail -4
for v in "$@"; do echo "== $v"; TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so python tools/p2v_time.py 2>&1 | tail -4; done
