mkdir -p gpurun_out
for v in new old; do
  if [ $v = old ]; then export TEXFORGE_CUDA_LIB=$PWD/tools/ab/libtexforge_cuda_old.so; else unset TEXFORGE_CUDA_LIB; fi
  for wl in c2 c4 c5; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b27_${v}_$wl.json 2>/dev/null; done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest27.log 2>&1
