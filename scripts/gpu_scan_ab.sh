#!/bin/bash
# Replay change check: every replay parity test, then the C5 sweep + shard proxy, main vs VARIANT (twice)
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_gpu_replay.py tests/test_gpu_replay_seg.py tests/test_gpu_replay_full.py \
  tests/test_gpu_policy.py tests/test_gpu_alg1.py tests/test_gpu_feedback.py tests/test_gpu_dist_shared.py \
  > gpurun_out/scan_tests.log 2>&1; echo "rc=$?" >> gpurun_out/scan_tests.log
run() { echo "== $1" >> gpurun_out/scan_ab.log; shift; timeout 900 "$@" >> gpurun_out/scan_ab.log 2>&1; }
for r in 1 2; do
  run "main" python bench.py --only-replay --replay-reps 3 --no-policies
  run "variant" env ORLOJ_LIB=$VARIANT python bench.py --only-replay --replay-reps 3 --no-policies
done
echo alldone >> gpurun_out/scan_ab.log
