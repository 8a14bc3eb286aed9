mkdir -p gpurun_out
timeout 300 python tools/e2e_diag.py > gpurun_out/e2e11.json 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b11_c3.json 2> gpurun_out/b11_c3.err
