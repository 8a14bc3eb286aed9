# Parity of the early per-band D2H + c3 bench e2e (run under gpurun).
mkdir -p gpurun_out/early
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/early/parity.log 2>&1; echo "rc=$?" >> gpurun_out/early/parity.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/early/bench_c3_$i.json 2> gpurun_out/early/bench_c3_$i.err; done
