#!/bin/bash
# Priority scores / PopBatch: parity tests, the P1 bench leg and one ncu --set
# full capture of each kernel.  Everything lands in gpurun_out/.
mkdir -p gpurun_out
[ -n "${SKIP_TESTS}" ] || timeout 600 python -m pytest tests/test_gpu_priority.py -q > gpurun_out/pytest_priority.log 2>&1 && echo "pytest rc=0" >> gpurun_out/pytest_priority.log
P1='import bench, torch, json; print(json.dumps(bench.run_priority(torch.device("cuda", 0), lambda x: x, 1)))'
timeout 300 python -c "$P1" > gpurun_out/bench_priority.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_priority.log
if [ -z "${SKIP_NCU}" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"priority_scores|pop_batch" -s 6 -c 2 -f \
   -o gpurun_out/prof_priority python -c "$P1" > gpurun_out/ncu_priority.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_priority.log
fi
