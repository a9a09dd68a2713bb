#!/bin/bash
# C2-HBM (per-request rows) with the main library and VARIANTS: score tests, then the bench leg twice each
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_score.py tests/test_gpu_guards.py tests/test_gpu_variants.py > gpurun_out/c2hbm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c2hbm_tests.log
C='import bench, torch, json; print(json.dumps(bench.run_c2_hbm(torch.device("cuda", 0), lambda x: x, 1, None)))'
for r in 1 2; do for v in "" ${VARIANTS}; do
  echo "== ${v:-main}" >> gpurun_out/c2hbm_ab.log
  ORLOJ_LIB=$v timeout 300 python -c "$C" >> gpurun_out/c2hbm_ab.log 2>&1
done; done
