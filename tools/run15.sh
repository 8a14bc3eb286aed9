mkdir -p gpurun_out
for v in new old; do
  if [ $v = old ]; then export TEXFORGE_CUDA_LIB=$PWD/tools/ab/libtexforge_cuda_old.so; else unset TEXFORGE_CUDA_LIB; fi
  for L in 256 128; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > gpurun_out/t15_${v}_L$L.json 2>&1; done
done
