#!/bin/bash
# iteration check: replay + score GPU tests, replay sweep timing + launch list, C2/C4 timing + ncu
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_replay.py tests/test_gpu_replay_seg.py tests/test_gpu_policy.py \
  tests/test_gpu_feedback.py tests/test_gpu_alg1.py tests/test_gpu_invariants.py tests/test_gpu_score.py \
  > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
timeout 600 python bench.py --only-replay --no-policies ${BARGS} > gpurun_out/replay_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
  -k regex:replay_kernel --log-file gpurun_out/replay_sweep_launches.csv \
  python bench.py --only-replay --replay-reps 1 --no-policies --no-shard-proxy > gpurun_out/ncu_sweep.log 2>&1
python scripts/c4_prof.py C4 4 > gpurun_out/c4_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_small -s 2 -c 1 -f \
  -o gpurun_out/prof_c4 python scripts/c4_prof.py C4 3 > gpurun_out/ncu_c4.log 2>&1
