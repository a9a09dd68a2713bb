#!/bin/bash
# A/B the pick kernel across library variants (ORLOJ_LIB) on the C3 bench loop.
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/variants.log
  ORLOJ_LIB=$v timeout 300 python bench.py --ncu --steps 50 --warmup 3 >> gpurun_out/variants.log 2>&1
done
