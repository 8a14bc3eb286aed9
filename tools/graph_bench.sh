# Bench workloads with and without the CUDA-graph step replay (run under gpurun).
mkdir -p gpurun_out/graph
for w in c1 c2 c4 c5; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --cpu-seconds 3 > gpurun_out/graph/g_$w.json 2> gpurun_out/graph/g_$w.err
  TFG_BENCH_GRAPH=0 timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/graph/e_$w.json 2> gpurun_out/graph/e_$w.err
done
timeout 900 python -m pytest tests/test_bench_dist.py -q -m gpu > gpurun_out/graph/bench_dist.log 2>&1; echo "rc=$?" >> gpurun_out/graph/bench_dist.log
