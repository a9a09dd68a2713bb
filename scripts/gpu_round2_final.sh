#!/bin/bash
# Round-2 evidence refresh on the committed code: smoke, GPU tests (parity stats),
# default bench line, reference arm, C3 launch list + ncu --set full of the pick,
# the replay sweep's instruction count + ncu of its first pass, and ncu of the
# C4 short-queue, priority / PopBatch and model-variant kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt
bash scripts/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --ncu --steps 5 --warmup 3 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 -f \
   -o gpurun_out/prof_c3_pick python bench.py --ncu --steps 3 --warmup 3 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
  -k regex:replay_kernel --log-file gpurun_out/replay_sweep_launches.csv \
  python bench.py --only-replay --replay-reps 1 --no-policies --no-shard-proxy > gpurun_out/ncu_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 4 -c 1 -f \
   -o gpurun_out/prof_replay python bench.py --only-replay --no-shard-proxy --no-policies --replay-seeds 64 \
   --replay-arrivals 20000 --replay-reps 1 > gpurun_out/ncu_replay.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_small -s 2 -c 1 -f \
   -o gpurun_out/prof_c4 python scripts/c4_prof.py C4 3 > gpurun_out/ncu_c4.log 2>&1
SKIP_TESTS=1 bash scripts/gpu_priority_prof.sh
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:model --log-file gpurun_out/model_launches.csv python scripts/model_variants_prof.py > gpurun_out/ncu_model.log 2>&1
python scripts/model_instr.py gpurun_out/model_launches.csv gpurun_out/model_variants_instr.json > gpurun_out/model_instr.log 2>&1
ORLOJ_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_shared.log 2>&1; echo "n2 rc=$?" >> gpurun_out/bench_n2_shared.log
echo done > gpurun_out/final_done.txt
