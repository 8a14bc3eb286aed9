mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest13.log 2>&1; echo "rc=$?" >> gpurun_out/pytest13.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b13_c3.json 2> gpurun_out/b13_c3.err
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b13_c4.json 2> gpurun_out/b13_c4.err
