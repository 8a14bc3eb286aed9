#!/bin/bash
# One GPU session: environment facts, microbenchmarks, parity tests, bench.
# Usage (under gpurun): bash tools/gpu_run.sh [stage...]; outputs in gpurun_out/
mkdir -p gpurun_out
OUT=gpurun_out
stages="${@:-info atomics smoke pytest bench}"
for s in $stages; do
  case $s in
    info)
      { nproc; lscpu | grep -E 'Model name|^CPU\(s\)|Thread|Socket'; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv; } > $OUT/info.txt 2>&1 ;;
    atomics)
      timeout 120 ./tools/atomics_bench > $OUT/atomics.json 2>&1 ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log ;;
    pytest)
      timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log ;;
    bench)
      timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err ;;
    benchref)
      timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err ;;
  esac
done
