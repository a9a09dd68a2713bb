#!/bin/bash
# A/B library variants (ORLOJ_LIB).  MODE=pick (C3 pick loop) or MODE=replay (C5 sweep).
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/variants.log
  if [ "${MODE:-pick}" = "replay" ]; then
    ORLOJ_LIB=$v timeout 600 python bench.py --only-replay --replay-reps 2 ${REPLAY_ARGS} >> gpurun_out/variants.log 2>&1
  else
    ORLOJ_LIB=$v timeout 300 python bench.py --ncu --steps 50 --warmup 3 >> gpurun_out/variants.log 2>&1
  fi
done
