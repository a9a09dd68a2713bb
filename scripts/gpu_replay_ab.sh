#!/bin/bash
# Replay A/B: segmented-replay parity tests, then the C5 sweep + 2/4/8 shard proxy for each
# spec in $SPECS ("label:ENV=VAL,ENV=VAL" ; ORLOJ_LIB=... selects a variant library).
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_replay_seg.py tests/test_gpu_replay_full.py tests/test_gpu_dist_shared.py \
  > gpurun_out/replay_ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/replay_ab_tests.log
for spec in $SPECS; do
  label=${spec%%:*}; envs=${spec#*:}
  echo "== $label" >> gpurun_out/replay_ab.log
  env ${envs//,/ } timeout 900 python bench.py --only-replay --replay-reps 3 --no-policies ${REPLAY_ARGS} >> gpurun_out/replay_ab.log 2>&1
done
echo alldone >> gpurun_out/replay_ab.log
