#!/bin/bash
# ncu --set full (+ SASS source page) of one vote launch for several libs.
# Usage: bash tools/r02_ncu_ab.sh TAG "lib1 lib2" L kind d:theta
O=gpurun_out/ncu_$1; mkdir -p $O
for lib in $2; do
  if [ $lib = cur ]; then unset TEXFORGE_CUDA_LIB; else export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_$lib.so; fi
  out=$O/${lib}_L$3_$4_${5/:/_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote -c 1 -f -o $out \
    python tools/profile_vote.py --levels $3 --kinds $4 --dts $5 --reps 1 > $out.log 2>&1
  ncu -i $out.ncu-rep --page raw --csv 2>/dev/null | gzip > $out.raw.csv.gz
  ncu -i $out.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $out.sass.csv.gz
  ncu -i $out.ncu-rep --page details 2>/dev/null > $out.details.txt
  rm -f $out.ncu-rep
done
