#!/bin/bash
# Build libgbx with extra nvcc defines into paper_2104_01661_b200/_variants/libgbx_NAME.so
# (for A/B sweeps on the GPU box: GBX_LIB=<path> selects it).
#   tools/build_variant.sh b0ipl8 "-DGBX_PR_B0IPL=8" pagerank
set -e
NAME=$1; FLAGS=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2104_01661_b200/csrc
OUT=$ROOT/paper_2104_01661_b200/_variants
mkdir -p $OUT/$NAME
make -s -C $C >/dev/null
objs=""
SRCS=$(sed -n "s/^SRCS := //p" $C/Makefile | sed "s/\.cu//g")
for f in $SRCS; do
  if [[ " $* " == *" $f "* ]]; then
    /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
      -Xcompiler -fPIC --expt-relaxed-constexpr -I$ROOT/include $FLAGS -c $C/$f.cu -o $OUT/$NAME/$f.o
    objs="$objs $OUT/$NAME/$f.o"
  else
    objs="$objs $ROOT/paper_2104_01661_b200/_build/$f.o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libgbx_$NAME.so $objs \
  -lcudart_static -lrt -lpthread -ldl
echo $OUT/libgbx_$NAME.so
