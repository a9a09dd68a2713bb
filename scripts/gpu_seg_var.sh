#!/bin/bash
# Segment-count sweep for several library variants (ORLOJ_LIB).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_replay_seg.py -q -x > gpurun_out/pytest_seg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_seg.log
for v in main e1 e4; do
  lib=""; [ $v != main ] && lib=build_variants/liborloj_$v.so
  ORLOJ_LIB=$lib timeout 900 python bench.py --replay-seg-sweep --replay-reps 2 --seg-sweep-n 1,8 --seg-sweep-g ${SEG_G:-1,8,16,32} > gpurun_out/seg_sweep_$v.log 2>&1
done
