#!/bin/bash
O=gpurun_out/walk_$1; mkdir -p $O
for L in $2; do
  TEXFORGE_WALK=0 timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/old_L$L.json 2>&1
  for lib in cur $3; do
    if [ $lib = cur ]; then unset TEXFORGE_CUDA_LIB; else export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_$lib.so; fi
    timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/${lib}_L$L.json 2>&1
  done
  unset TEXFORGE_CUDA_LIB
done
[ -n "$4" ] && { timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$4" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; }
true
