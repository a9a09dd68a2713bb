#!/bin/bash
# PopBatch change check: priority parity + guard tests, then the P1 leg with the main library and VARIANTS (twice each)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_priority.py tests/test_gpu_guards.py > gpurun_out/pop_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pop_tests.log
VARIANTS="$VARIANTS" bash scripts/gpu_prio_var.sh
echo done >> gpurun_out/prio_var.log
