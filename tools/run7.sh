mkdir -p gpurun_out
for v in new old; do
  if [ $v = old ]; then export TEXFORGE_CUDA_LIB=$PWD/tools/ab/libtexforge_cuda_old.so; else unset TEXFORGE_CUDA_LIB; fi
  for L in 256 32; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > gpurun_out/t7_${v}_L$L.json 2>&1; done
done
unset TEXFORGE_CUDA_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o gpurun_out/prof7_L32 python tools/profile_vote.py --levels 32 --kinds noise --reps 1 > gpurun_out/ncu7.log 2>&1
