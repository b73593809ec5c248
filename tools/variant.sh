#!/bin/bash
# Build a variant library: tools/variant.sh NAME "-DFLAG ..." [src.cu ...]
# Recompiles the named sources (default tc_fwd.cu) with the extra flags, reuses the
# other objects of the main build, links var/libadattn_b200_NAME.so (dev tool).
set -e
NAME=$1; FLAGS=$2; shift 2
SRCS=${@:-tc_fwd.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
P=$ROOT/paper_2604_15180_b200
OUT=$ROOT/var/$NAME; mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -fmad=false -I$ROOT/include -I$P/csrc --expt-relaxed-constexpr"
OBJS=""
for o in $P/build/*.o; do
  b=$(basename $o .o)
  if echo " $SRCS " | grep -q " $b.cu "; then
    $NV $FLAGS -c $P/csrc/$b.cu -o $OUT/$b.o
    OBJS="$OBJS $OUT/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/var/libadattn_b200_$NAME.so $OBJS -lcudart -lcuda
echo built var/libadattn_b200_$NAME.so
