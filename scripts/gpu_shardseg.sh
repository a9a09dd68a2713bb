#!/bin/bash
# 8-GPU shard proxy for several segment specs (bench --proxy-segments)
mkdir -p gpurun_out
for spec in ${SPECS}; do
  echo "== $spec" >> gpurun_out/shardseg.log
  timeout 900 python bench.py --only-replay --replay-reps 3 --no-policies --proxy-segments "$spec" >> gpurun_out/shardseg.log 2>&1
done
echo alldone >> gpurun_out/shardseg.log
