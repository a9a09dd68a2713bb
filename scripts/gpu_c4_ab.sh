#!/bin/bash
# C4 / C2 timing of the main library and variant libraries (ORLOJ_LIB), twice each
mkdir -p gpurun_out
for r in 1 2; do for v in "" ${VARIANTS}; do
  echo "== ${v:-main}" >> gpurun_out/c4_ab.log
  ORLOJ_LIB=$v python scripts/c4_prof.py C4 4 >> gpurun_out/c4_ab.log 2>&1
  ORLOJ_LIB=$v python scripts/c4_prof.py C2 4 >> gpurun_out/c4_ab.log 2>&1
done; done
