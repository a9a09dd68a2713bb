#!/bin/bash
# Replay drain experiments: segments of the last-launched family (bench --replay-segments / --proxy-segments "auto,last=...")
mkdir -p gpurun_out
run() { echo "== $1" >> gpurun_out/lastseg.log; shift; timeout 900 "$@" >> gpurun_out/lastseg.log 2>&1; }
B="python bench.py --only-replay --replay-reps 3 --no-policies"
run "base" $B
run "last x2" $B --replay-segments "auto,last=x2" --proxy-segments "auto,last=x2"
run "last x3" $B --replay-segments "auto,last=x3" --proxy-segments "auto,last=x3"
run "last x2 tail0" env ORLOJ_SEG_TAIL=0 $B --replay-segments "auto,last=x2" --proxy-segments "auto,last=x2"
run "all 48" $B --proxy-segments 48 --no-shard-proxy
run "proxy 48" $B --proxy-segments 48
run "proxy 32 last 64" $B --proxy-segments "32,last=64"
echo alldone >> gpurun_out/lastseg.log
