#!/bin/bash
# Launch list (time, instructions, warps active) of each family's rank-0 shard of 8 GPUs at several segment counts
mkdir -p gpurun_out
for G in 24 48; do
for fam in skipnet rdi gpt static; do
DIAG_WORLD=8 DIAG_ARRIVALS=100000 DIAG_SEGMENTS=$G DIAG_FAMILY=$fam timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:replay_kernel --log-file gpurun_out/shard8_${fam}_g$G.csv python scripts/replay_one_family.py > /dev/null 2>&1
done
done
