#!/bin/bash
# ncu --set full of the segmented replay's first pass (MODE 1) on one full C5 family + launch list of the sweep
mkdir -p gpurun_out
DIAG_WORLD=1 DIAG_ARRIVALS=100000 DIAG_SEGMENTS=8 DIAG_FAMILY=${FAM:-skipnet} timeout 900 ncu --set full --clock-control none \
  --import-source on -k regex:replay_kernel -c 2 -f -o gpurun_out/prof_replay_${FAM:-skipnet} \
  python scripts/replay_one_family.py > gpurun_out/ncu_replay.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_replay.log
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
  -k regex:replay_kernel --log-file gpurun_out/replay_sweep_launches.csv \
  python bench.py --only-replay --replay-reps 1 --no-policies --no-shard-proxy > gpurun_out/ncu_sweep.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/ncu_sweep.log
