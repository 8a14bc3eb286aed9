#!/bin/bash
O=gpurun_out/ab2; mkdir -p $O
run() { # name levels
  timeout 300 python tools/profile_vote.py --levels $2 --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/$1_L$2.json 2>&1; }
for L in 256 32 64; do
  TEXFORGE_ALIGN=0 run unaligned $L
  run aligned $L
  TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_cg.so run cg $L
  TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_noalloc.so run noalloc $L
done
for v in base noret; do
  if [ $v = base ]; then unset TEXFORGE_CUDA_LIB; else export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_$v.so; fi
  timeout 600 ncu --set full --clock-control none -k regex:glcm_vote -c 1 -f -o $O/ncu_$v python tools/profile_vote.py --levels 256 --kinds noise --dts 1:0 --reps 1 > /dev/null 2>&1
  ncu -i $O/ncu_$v.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/ncu_${v}_raw.csv.gz
  ncu -i $O/ncu_$v.ncu-rep --page details 2>/dev/null > $O/ncu_${v}_details.txt
  rm -f $O/ncu_$v.ncu-rep
done
unset TEXFORGE_CUDA_LIB
timeout 600 ncu --set full --clock-control none -k regex:bench -f -o $O/ncu_atom ./tools/atomics_bench > /dev/null 2>&1
ncu -i $O/ncu_atom.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/ncu_atom_raw.csv.gz; rm -f $O/ncu_atom.ncu-rep
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
