export PYTHONPATH=$PWD
for v in "$@"; do TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$v.so timeout 120 python tools/k1_ab.py cube6 8 7 2>&1 | tail -1 | sed "s/^/$v /"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"p1_pipe" -c 1 python tools/k1_ab.py cube6 8 7 2>&1 | grep -E "duration|bytes|inst_exec|warps_active"
