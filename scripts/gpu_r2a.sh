#!/bin/bash
# round 2: GPU tests + functional 2-rank self-launch + full bench line
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/host.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
ORLOJ_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --queues 8192 --no-extra --no-e2e \
  --no-policies --replay-seeds 32 --replay-arrivals 20000 > gpurun_out/bench_n2_selflaunch.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_selflaunch.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
