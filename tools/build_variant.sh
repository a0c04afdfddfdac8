#!/bin/bash
# Build a variant of libtetmf_b200.so with one kernel source recompiled under
# extra -D flags (tuning sweeps). Usage:
#   tools/build_variant.sh NAME SOURCE.cu "-DFOO=1 -DBAR=2"
# Output: paper_2404_08371_b200/_lib/variants/libtetmf_NAME.so (select with TETMF_LIB)
set -e
NAME=$1; SRC=$2; DEFS=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_2404_08371_b200/csrc
LIB=$ROOT/paper_2404_08371_b200/_lib
NCCL_DIR=$(python -c "import nvidia.nccl as n; print(list(n.__path__)[0])")
OUT=$LIB/variants; mkdir -p $OUT/$NAME
make -s -C $CSRC -j8 >/dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Xptxas -v,-warn-spills -I$NCCL_DIR/include $DEFS \
  -c $CSRC/$SRC -o $OUT/$NAME/${SRC%.cu}.o 2> $OUT/$NAME/ptxas.log
OBJS=$(ls $LIB/obj/*.o | grep -v "/${SRC%.cu}.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libtetmf_$NAME.so $OBJS $OUT/$NAME/${SRC%.cu}.o \
  -L$NCCL_DIR/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL_DIR/lib -lcudart -lpthread
grep -E "registers|spill" $OUT/$NAME/ptxas.log | grep -B1 -A0 "registers" | head -20 | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | paste -sd' ' | sed "s/^/$NAME: /"
