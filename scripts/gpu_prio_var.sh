#!/bin/bash
# P1 priority leg with variant libraries (ORLOJ_LIB) built with extra -D flags
mkdir -p gpurun_out
P1='import bench, torch, json; print(json.dumps(bench.run_priority(torch.device("cuda", 0), lambda x: x, 1)))'
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then lib=""; else lib=$PWD/build_variants/lib_$v.so; fi
  for rep in 1 2; do
    ORLOJ_LIB=$lib timeout 300 python -c "$P1" 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['ms_scores'], d['ms_pop'])" >> gpurun_out/prio_var.log 2>&1
  done
done
