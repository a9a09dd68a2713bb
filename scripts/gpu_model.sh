#!/bin/bash
# Scoring-model variants: parity tests, the C2 variant timings, the ncu launch
# list of one launch per variant (instructions for the issue roofline)
mkdir -p gpurun_out
timeout 600 python -m pytest -q tests/test_gpu_variants.py > gpurun_out/pytest_model.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_model.log
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:model --log-file gpurun_out/model_launches.csv python scripts/model_variants_prof.py > gpurun_out/ncu_model.log 2>&1
python scripts/model_instr.py gpurun_out/model_launches.csv gpurun_out/model_variants_instr.json > gpurun_out/model_instr.log 2>&1 && cp gpurun_out/model_variants_instr.json profiles/
M='import bench, torch, json; print(json.dumps(bench.run_model_variants(torch.device("cuda", 0), lambda x: x, 1)))'
timeout 300 python -c "$M" > gpurun_out/bench_model.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_model.log
