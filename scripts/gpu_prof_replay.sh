#!/bin/bash
mkdir -p gpurun_out
DIAG_WORLD=1 DIAG_ARRIVALS=100000 DIAG_SEGMENTS=8 DIAG_FAMILY=${FAM:-skipnet} timeout 900 ncu --set full --clock-control none \
  --import-source on -k regex:replay_kernel -c 1 -f -o gpurun_out/prof_replay_${FAM:-skipnet} \
  python scripts/replay_one_family.py > gpurun_out/ncu_replay.log 2>&1
