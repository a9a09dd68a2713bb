#!/bin/bash
# 1-GPU C5 sweep for several segment specs (bench --replay-segments), no shard proxy
mkdir -p gpurun_out
for spec in ${SPECS}; do
  echo "== $spec" >> gpurun_out/sweepseg.log
  timeout 900 python bench.py --only-replay --replay-reps 3 --no-policies --no-shard-proxy --replay-segments "$spec" >> gpurun_out/sweepseg.log 2>&1
done
echo alldone >> gpurun_out/sweepseg.log
