#!/bin/bash
O=gpurun_out/jobs_$1; mkdir -p $O
for sz in 4096 2048 512; do for L in 8 16 32 64; do
  for j in 0 1; do
    TEXFORGE_JOBS=$j timeout 300 python tools/profile_vote.py --size $sz --levels $L --dts 1:0,1:45,1:90,1:135 --reps 7 --multi --time > $O/jobs${j}_${sz}_L$L.json 2>&1
  done
done; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
