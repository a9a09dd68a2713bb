#!/bin/bash
# Short-queue kernel check: its parity tests, C4/C2 A/B against VARIANTS, ncu of the C4 pick
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_score.py tests/test_gpu_invariants.py tests/test_gpu_variants.py > gpurun_out/c4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c4_tests.log
VARIANTS="${VARIANTS}" bash scripts/gpu_c4_ab.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_small -s 2 -c 1 -f \
   -o gpurun_out/prof_c4 python scripts/c4_prof.py C4 3 > gpurun_out/ncu_c4.log 2>&1
echo done >> gpurun_out/c4_ab.log
