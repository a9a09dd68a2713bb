#!/bin/bash
# Replay A/B: scenario order in the trace (seed groups vs SLO bucket by bucket), persistent first pass
mkdir -p gpurun_out
run() { echo "== $1" >> gpurun_out/order_ab.log; shift; timeout 900 "$@" >> gpurun_out/order_ab.log 2>&1; }
B="python bench.py --only-replay --replay-reps 3 --no-policies"
L="--replay-segments auto,last=x2 --proxy-segments auto,last=x2"
run "seed last2" $B $L
run "bucket last2" $B $L --scenario-order bucket
run "bucket persist last2" env ORLOJ_LIB=build_variants/liborloj_persist.so $B $L --scenario-order bucket
run "bucket" $B --scenario-order bucket
run "seed last2 again" $B $L
echo alldone >> gpurun_out/order_ab.log
