#!/bin/bash
# Short-queue kernel (C2/C4): score parity tests, timing, one ncu --set full capture of the C4 pick
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_score.py tests/test_gpu_invariants.py > gpurun_out/pytest_score.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_score.log
python scripts/c4_prof.py C4 4 > gpurun_out/c4_time.log 2>&1
python scripts/c4_prof.py C2 4 >> gpurun_out/c4_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_small -s 2 -c 1 -f \
  -o gpurun_out/prof_c4 python scripts/c4_prof.py C4 3 > gpurun_out/ncu_c4.log 2>&1
