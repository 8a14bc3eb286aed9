#!/bin/bash
# A/B over sizes: bash tools/r02_abs.sh TAG "libs" "levels" "sizes" [pytest -k]
O=gpurun_out/abs_$1; mkdir -p $O
for lib in $2; do
  if [ $lib = cur ]; then unset TEXFORGE_CUDA_LIB; else export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_$lib.so; fi
  for L in $3; do for sz in $4; do
    timeout 300 python tools/profile_vote.py --size $sz --levels $L --dts 1:0,1:45,2:90,4:135 --reps 7 --time > $O/${lib}_L${L}_s$sz.json 2>&1
  done; done
done
unset TEXFORGE_CUDA_LIB
if [ -n "$5" ]; then timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$5" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; fi
true
