#!/bin/bash
# replay changes: replay GPU tests, the timed C5 sweep (+ shard proxy), and the sweep's warp-instruction count
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_replay.py tests/test_gpu_replay_seg.py tests/test_gpu_policy.py \
  tests/test_gpu_feedback.py tests/test_gpu_replay_full.py tests/test_gpu_alg1.py tests/test_gpu_invariants.py \
  > gpurun_out/pytest_replay.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_replay.log
timeout 600 python bench.py --only-replay --no-policies ${BARGS} > gpurun_out/replay_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
  -k regex:replay_kernel --log-file gpurun_out/replay_sweep_launches.csv \
  python bench.py --only-replay --replay-reps 1 --no-policies --no-shard-proxy > gpurun_out/ncu_sweep.log 2>&1
