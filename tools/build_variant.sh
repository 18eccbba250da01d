#!/bin/bash
# build_variant.sh NAME "EXTRA NVCC FLAGS" -> tools/exp/libfek_NAME.so (QSS-only experiment build)
set -e
NAME=$1; FLAGS=$2
ROOT=${ROOT:-/root/repo}; CS=$ROOT/paper_1504_01023_b200/csrc; OUT=$ROOT/build/exp_$NAME
mkdir -p $OUT $ROOT/tools/exp
for src in $CS/fek_abi.cu $CS/fek_mesh.cu $CS/fek_layout.cu $CS/cases/*.cu; do
  b=$(basename $src .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 --fmad=false -Xcompiler -fPIC -I$ROOT/include -DFEK_QSS_ONLY -DFEK_NO_TILES $FLAGS -c $src -o $OUT/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static $OUT/*.o -o $ROOT/tools/exp/libfek_$NAME.so
echo built $NAME
