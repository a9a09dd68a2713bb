#!/bin/bash
# ncu launch lists (time, warp instructions, warps active, issue active) of the rank-0 shard of 8 and of 1
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for spec in ${SPECS:-"8:auto" "8:48" "1:auto"}; do
  W=${spec%%:*}; G=${spec#*:}
  WORLD=$W SEGS=$G timeout 900 ncu --metrics $M --clock-control none --csv -k regex:replay_kernel \
    --log-file gpurun_out/shard_w${W}_g${G}.csv python scripts/shard_once.py > gpurun_out/shard_w${W}_g${G}.log 2>&1
done
echo done > gpurun_out/shard_ncu_done.txt
