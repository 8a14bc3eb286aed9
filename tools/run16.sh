mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest16.log 2>&1
for v in new old; do
  if [ $v = old ]; then export TEXFORGE_CUDA_LIB=$PWD/tools/ab/libtexforge_cuda_old.so; else unset TEXFORGE_CUDA_LIB; fi
  for L in 32 64; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > gpurun_out/t16_${v}_L$L.json 2>&1; done
  timeout 300 python tools/profile_vote.py --size 4096 --levels 32 --dts 1:0,1:45,2:90,4:135 --reps 5 --time > gpurun_out/t16_${v}_small.json 2>&1
  timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b16_${v}_c2.json 2>/dev/null
done
