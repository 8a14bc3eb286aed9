# Self-re-arming cooperative counters: GPU parity + c3 bench + launch list (run under gpurun).
mkdir -p gpurun_out/rearm
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/rearm/parity.log 2>&1; echo "rc=$?" >> gpurun_out/rearm/parity.log
for i in 1 2; do timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rearm/bench_c3_$i.json 2> gpurun_out/rearm/bench_c3_$i.err; done
