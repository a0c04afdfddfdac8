export PYTHONPATH=$PWD
for v in copyonly copyonlyr16 copyonlyc128; do
TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"p1_smem" -c 1 python tools/k1_ab.py cube6 8 0 2>/dev/null | grep -E "duration|bytes_read" | sed "s/^/$v /"
done
