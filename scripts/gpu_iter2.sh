#!/bin/bash
# C4 timing; replay source profile (full C5 skipnet, 8 segments); 8-GPU rank-0 shard launch list per family
mkdir -p gpurun_out
timeout 300 python -m pytest -q -x tests/test_gpu_score.py -k "config4 or config2 or config1" > gpurun_out/pytest_c4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c4.log
python scripts/c4_prof.py C4 4 > gpurun_out/c4_time.log 2>&1
DIAG_WORLD=1 DIAG_ARRIVALS=100000 DIAG_SEGMENTS=8 DIAG_FAMILY=skipnet timeout 900 ncu --set full --clock-control none \
  --import-source on -k regex:replay_kernel -c 1 -f -o gpurun_out/prof_replay_skipnet \
  python scripts/replay_one_family.py > gpurun_out/ncu_replay.log 2>&1
for fam in skipnet rdi gpt static; do
DIAG_WORLD=8 DIAG_ARRIVALS=100000 DIAG_SEGMENTS=24 DIAG_FAMILY=$fam timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:replay_kernel --log-file gpurun_out/shard8_$fam.csv python scripts/replay_one_family.py > /dev/null 2>&1
done
