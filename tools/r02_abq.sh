#!/bin/bash
# A/B of tools/ab/lib_*.so variants (and the in-tree lib as "cur"): per-(d,theta) rates.
# Usage: bash tools/r02_abq.sh TAG "cur lib1 lib2" "levels" [dts]
O=gpurun_out/abq_$1; mkdir -p $O
dts=${4:-1:0,1:45,1:90,1:135}
for lib in $2; do
  if [ $lib = cur ]; then unset TEXFORGE_CUDA_LIB; else export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_$lib.so; fi
  for L in $3; do timeout 300 python tools/profile_vote.py --levels $L --dts $dts --reps 5 --time > $O/${lib}_L$L.json 2>&1; done
done
