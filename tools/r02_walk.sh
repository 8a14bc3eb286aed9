#!/bin/bash
O=gpurun_out/walk_$1; mkdir -p $O
for L in $2; do
  TEXFORGE_WALK=0 timeout 300 python tools/profile_vote.py --levels $L --dts ${3:-1:0,1:45,1:90,1:135} --reps 5 --time > $O/old_L$L.json 2>&1
  timeout 300 python tools/profile_vote.py --levels $L --dts ${3:-1:0,1:45,1:90,1:135} --reps 5 --time > $O/walk_L$L.json 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${4:-parity}" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
