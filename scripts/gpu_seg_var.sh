#!/bin/bash
# Segment-count sweep for several library variants (ORLOJ_LIB); VARIANTS="main e1 ..."
mkdir -p gpurun_out
for v in ${VARIANTS:-main}; do
  lib=""; [ $v != main ] && lib=build_variants/liborloj_$v.so
  ORLOJ_LIB=$lib timeout 900 python bench.py --replay-seg-sweep --replay-reps 2 --seg-sweep-n ${SEG_N:-1,8} --seg-sweep-g ${SEG_G:-auto} > gpurun_out/seg_sweep_$v.log 2>&1
done
