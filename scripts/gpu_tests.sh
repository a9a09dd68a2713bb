#!/bin/bash
# GPU test suite with parity statistics (tie counts, priority error vs the exact model) logged
mkdir -p gpurun_out
rm -f gpurun_out/parity_stats.jsonl
ORLOJ_PARITY_LOG=$PWD/gpurun_out/parity_stats.jsonl timeout ${T:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS} \
  > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
