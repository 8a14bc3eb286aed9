#!/bin/bash
O=gpurun_out/walk_$1; mkdir -p $O
for sz in 16384 4096; do for L in 32 256; do
  TEXFORGE_WALK=0 timeout 300 python tools/profile_vote.py --size $sz --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/old_${sz}_L$L.json 2>&1
  timeout 300 python tools/profile_vote.py --size $sz --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/walk_${sz}_L$L.json 2>&1
done; done
