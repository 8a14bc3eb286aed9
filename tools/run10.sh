mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest10.log 2>&1; echo "rc=$?" >> gpurun_out/pytest10.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/b10_c3.json 2> gpurun_out/b10_c3.err
timeout 300 python tools/e2e_diag.py > gpurun_out/e2e10.json 2>&1
for wl in c2 c4; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b10_$wl.json 2> gpurun_out/b10_$wl.err; done
