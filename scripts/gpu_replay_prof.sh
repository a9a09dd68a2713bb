#!/bin/bash
# Replay kernel: a timed sweep and one ncu --set full capture.
mkdir -p gpurun_out
timeout 600 python bench.py --only-replay --replay-seeds ${SEEDS:-256} --replay-reps 2 > gpurun_out/replay_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 4 -c 1 -f \
   -o gpurun_out/prof_replay python bench.py --only-replay --replay-seeds 32 --replay-arrivals 20000 --replay-reps 1 \
   > gpurun_out/ncu_replay.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_replay.log
