export PYTHONPATH=$PWD
timeout 120 python tools/k1_ab.py cube6 8 0 2>&1 | tail -1
TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_nost.so timeout 120 python tools/k1_ab.py cube6 8 0 2>&1 | tail -1 | sed "s/^/nost /"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"p1_smem|p1_face|interface" --csv python tools/k1_ab.py cube6 8 0 2>/dev/null | grep -E "p1_smem|p1_face|interface" | tail -3
