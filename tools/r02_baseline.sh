#!/bin/bash
# Round-2 session-start baseline (under gpurun): smoke, GPU suite, c3 bench,
# per-L kernel rates, one ncu capture of the L=256 noise vote kernel.
O=gpurun_out/r02b; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "rc=$?" >> $O/bench_c3.err
for L in 256 128 64 32; do
  timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/rates_L$L.json 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
