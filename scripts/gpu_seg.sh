#!/bin/bash
# Segmented replay: parity tests, then the segment-count sweep (full C5 and rank-0 shards).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_replay_seg.py tests/test_gpu_replay.py -q -x > gpurun_out/pytest_seg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_seg.log
timeout 1200 python bench.py --replay-seg-sweep --replay-reps 2 > gpurun_out/seg_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/seg_sweep.log
