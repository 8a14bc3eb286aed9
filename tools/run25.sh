mkdir -p gpurun_out
for rep in 1 2; do for v in new old; do
  if [ $v = old ]; then export TEXFORGE_CUDA_LIB=$PWD/tools/ab/libtexforge_cuda_old.so; else unset TEXFORGE_CUDA_LIB; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b25_${v}_$rep.json 2>/dev/null
done; done
