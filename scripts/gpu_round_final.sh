#!/bin/bash
# Full evidence run: smoke, GPU tests, default bench line, reference arm, launch
# list, ncu --set full on the C3 pick kernel, the segmented replay's first pass
# and the C4 short-queue kernel, and the replay segment sweep.
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
   -o gpurun_out/prof_replay python bench.py --only-replay --no-shard-proxy --no-policies --replay-seeds 64 \
   --replay-arrivals 20000 --replay-reps 1 > gpurun_out/ncu_replay.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_small -s 2 -c 1 -f \
   -o gpurun_out/prof_c4 python scripts/c4_prof.py C4 3 > gpurun_out/ncu_c4.log 2>&1
timeout 900 python bench.py --replay-seg-sweep --replay-reps 2 --seg-sweep-n 1,8 --seg-sweep-g 1,8,16,24,auto \
   > gpurun_out/seg_sweep.log 2>&1
echo done > gpurun_out/final_done.txt
