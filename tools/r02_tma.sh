#!/bin/bash
O=gpurun_out/tma; mkdir -p $O
for lib in base tma; do
  export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_$lib.so
  for L in 256 64 32; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/${lib}_L$L.json 2>&1; done
done
export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_tma.so
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "parity" > $O/pytest_tma.log 2>&1; echo "rc=$?" >> $O/pytest_tma.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote -c 1 -f -o $O/tma_L256_smooth python tools/profile_vote.py --levels 256 --kinds smooth --dts 1:0 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/tma_L256_smooth.ncu-rep --sass 20 > $O/tma_L256_smooth.txt 2>&1; rm -f $O/*.ncu-rep
