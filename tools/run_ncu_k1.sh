export PYTHONPATH=$PWD
# ncu captures of one K1 variant (arg 1) on cube6 L8: launch list + one full capture of each kernel
V=${1:-6}; LIB=${2:-}
[ -n "$LIB" ] && export TETMF_LIB=paper_2404_08371_b200/_lib/variants/libtetmf_$LIB.so
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"p1_" --csv \
  --log-file gpurun_out/k1_launches_v$V$LIB.csv python tools/k1_ab.py cube6 8 $V > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"p1_smem|p1_face|p1_interior|p1_stencil" -c 2 \
  -o gpurun_out/k1_full_v$V$LIB python tools/k1_ab.py cube6 8 $V > /dev/null 2>&1
echo done
