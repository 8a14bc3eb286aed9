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
    quick)
      for L in 256 32; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > $OUT/timing_L$L.json 2>&1; done ;;
    timing)
      for L in 256 64 32 16 8; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > $OUT/timing_L$L.json 2>&1; done
      for S in 1 2 3 4; do timeout 300 python tools/profile_vote.py --levels 32 --strategy $S --dts 1:0 --reps 5 --time > $OUT/timing_L32_s$S.json 2>&1; done
      for S in 3 4; do timeout 300 python tools/profile_vote.py --levels 128 --strategy $S --dts 1:0 --reps 5 --time > $OUT/timing_L128_s$S.json 2>&1; done ;;
    ncu)
      # exactly one timed step of the default bench: skip the 4 earlier steps (1 check + 3 warm-up) x 24 vote launches
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glcm -s 96 -c 24 --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_bench.json 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:glcm_ -c 4 -o $OUT/prof_c3 python tools/profile_vote.py --reps 1 --kinds noise,smooth > $OUT/ncu_full.log 2>&1 ;;
    ncu32)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o $OUT/prof_L32 python tools/profile_vote.py --levels 32 --kinds noise --reps 1 > $OUT/ncu_L32.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o $OUT/prof_L256 python tools/profile_vote.py --levels 256 --kinds noise --reps 1 > $OUT/ncu_L256.log 2>&1 ;;
    cpp)
      for b in dropin_tests refsuite_unit refsuite_accept; do timeout 900 tests/cpp/_build/$b > $OUT/cpp_$b.log 2>&1; echo "rc=$?" >> $OUT/cpp_$b.log; done ;;
    e2e)
      timeout 600 python tools/e2e_diag.py > $OUT/e2e_diag.json 2>&1 ;;
    benchref)
      timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err ;;
  esac
done
