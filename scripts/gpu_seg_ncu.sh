#!/bin/bash
# Per-kernel durations (ncu launch list, serialised) of the segmented replay at one shard size.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/seg_launches.csv \
  python bench.py --replay-seg-sweep --replay-reps 1 --seg-sweep-n ${SEG_N:-8} --seg-sweep-g ${SEG_G:-8,16,32} > gpurun_out/seg_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/seg_ncu.log
