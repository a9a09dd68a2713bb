#!/bin/bash
# Round-2 re-entry check: GPU tests with parity stats, smoke, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
bash scripts/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
echo done > gpurun_out/state_done.txt
