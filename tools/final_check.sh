# Final check of the session (run under gpurun): full GPU suite, smoke, c3 bench line.
mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
