#!/bin/bash
# Full evidence run: smoke, GPU tests, default bench line, launch list, ncu full on
# the pick kernel and on the replay kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --ncu --steps 5 --warmup 2 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 -f \
   -o gpurun_out/prof_c3_pick python bench.py --ncu --steps 3 --warmup 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 4 -c 1 -f \
   -o gpurun_out/prof_replay python bench.py --only-replay --no-shard-proxy --replay-seeds 64 --replay-arrivals 20000 \
   --replay-reps 1 > gpurun_out/ncu_replay.log 2>&1
echo done > gpurun_out/final_done.txt
