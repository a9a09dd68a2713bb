#!/bin/bash
# build_variant.sh NAME [nvcc -D flags...]: build liborloj into build_variants/ and
# print registers / spills of the C3 pick kernel and its SASS instruction mix.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/build_variants/liborloj_$NAME.so
mkdir -p $ROOT/build_variants
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v -shared -Xcompiler -fPIC "$@" \
  -o $OUT $ROOT/paper_2209_00159_b200/csrc/orloj.cu > /tmp/ptxas_$NAME.log 2>&1 || { grep -m5 error /tmp/ptxas_$NAME.log; exit 1; }
grep -A2 "score_kernelILi8ELi8ELb1ELb1" /tmp/ptxas_$NAME.log | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores"
cuobjdump -sass $OUT > /tmp/all_$NAME.sass
L=$(grep -n "Function : _ZN5orloj12score_kernelILi8ELi8ELb1ELb1E" /tmp/all_$NAME.sass | cut -d: -f1)
awk -v s=$L 'NR>=s' /tmp/all_$NAME.sass | awk 'NR>1 && /Function :/{exit} {print}' > /tmp/c3_$NAME.sass
echo "sass lines: $(grep -c '' /tmp/c3_$NAME.sass)"
