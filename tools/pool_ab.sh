# A/B of the shared tail pool: in-tree library at several TEXFORGE_POOL_PCT
# values vs tools/ab/lib_head.so (run under gpurun).
mkdir -p gpurun_out/pool
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pool/parity.txt
for cfg in ${POOL_CFGS:-head p0 p10 p20}; do
  if [ "${cfg#head}" != "$cfg" ]; then export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_head.so; unset TEXFORGE_POOL_PCT; else unset TEXFORGE_CUDA_LIB; export TEXFORGE_POOL_PCT=${cfg#p}; fi
  for L in 256 32; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 7 --time > gpurun_out/pool/${cfg}_L$L.json 2>&1; done
  for w in ${POOL_WORKLOADS:-c3 c4}; do timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/pool/${cfg}_$w.json 2>gpurun_out/pool/${cfg}_$w.err; done
done
