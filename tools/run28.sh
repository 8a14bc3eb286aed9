mkdir -p gpurun_out
for v in new old new old; do
  if [ $v = old ]; then export TEXFORGE_CUDA_LIB=$PWD/tools/ab/libtexforge_cuda_old.so; else unset TEXFORGE_CUDA_LIB; fi
  timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b28_${v}.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('gpurun_out/b28_${v}.json')); print('$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3))" >> gpurun_out/b28.txt
done
