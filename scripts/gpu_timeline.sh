#!/bin/bash
# Replay timeline diagnostics (scripts/replay_timeline.py) with the ORLOJ_REPLAY_TIMELINE variant
mkdir -p gpurun_out
export ORLOJ_LIB=build_variants/liborloj_timeline.so
for spec in ${SPECS:-"WORLD=8,RANK_=0" "WORLD=1"}; do
  echo "== $spec" >> gpurun_out/timeline.log
  env ${spec//,/ } timeout 600 python scripts/replay_timeline.py >> gpurun_out/timeline.log 2>&1
done
echo alldone >> gpurun_out/timeline.log
