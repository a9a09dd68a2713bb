#!/bin/bash
# Priority / PopBatch iteration: the priority, Alg. 1 and policy GPU tests (with
# parity stats), the P1 bench leg, one ncu --set full capture of each kernel.
mkdir -p gpurun_out
rm -f gpurun_out/parity_stats.jsonl
ORLOJ_PARITY_LOG=$PWD/gpurun_out/parity_stats.jsonl timeout 900 python -m pytest -q tests/test_gpu_priority.py \
  tests/test_gpu_alg1.py tests/test_gpu_policy.py > gpurun_out/pytest_priority.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_priority.log
SKIP_TESTS=1 bash scripts/gpu_priority_prof.sh
