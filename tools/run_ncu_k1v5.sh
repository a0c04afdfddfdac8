export PYTHONPATH=$PWD
# one full capture of the interior kernel and the face kernel (variant 5), cube6 L8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"p1_interior|p1_face" -c 2 \
  -o gpurun_out/k1v5_full python tools/k1_ab.py cube6 8 5 > gpurun_out/k1v5_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"p1_stencil2" -c 1 \
  -o gpurun_out/k1v2_full python tools/k1_ab.py cube6 8 0 >> gpurun_out/k1v5_ncu.log 2>&1
tail -3 gpurun_out/k1v5_ncu.log
