#!/bin/bash
# One GPU round: smoke, GPU tests, a bench line, the ncu launch list and one
# ncu --set full capture of the pick kernel.  Everything lands in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -z "${SKIP_NCU}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --ncu --steps 5 --warmup 2 > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 -f \
   -o gpurun_out/prof_c3_pick python bench.py --ncu --steps 3 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/ncu_full.log
fi
