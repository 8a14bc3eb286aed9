# Full round evidence pass (run under gpurun): smoke, pytest -m gpu, C++ drop-in + reference suites,
# CLI suite, bench (all BASELINE configs + reference arm), one-step ncu launch list, ncu --set full
# summaries of the vote kernel, per-L kernel rates. Outputs in gpurun_out/r14/ (see profiles/README.md).
mkdir -p gpurun_out/r14
O=gpurun_out/r14
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/info.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for b in dropin_tests refsuite_unit refsuite_accept; do timeout 900 tests/cpp/_build/$b > $O/cpp_$b.log 2>&1; echo "rc=$?" >> $O/cpp_$b.log; done
TEXFORGE_CLI=$PWD/cli/_build/texforge timeout 900 cli/_build/refsuite_cli > $O/cli_refsuite.log 2>&1; echo "rc=$?" >> $O/cli_refsuite.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --impl reference > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
for wl in c2 c4 c5 c1; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --cpu-seconds 5 > $O/bench_$wl.json 2> $O/bench_$wl.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glcm -s 96 -c 24 --csv --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
for K in noise smooth; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o /tmp/full_$K python tools/profile_vote.py --levels 256 --kinds $K --reps 1 > $O/ncu_full_$K.log 2>&1
  python tools/ncu_summary.py /tmp/full_$K.ncu-rep > $O/ncu_vote_L256_$K.txt 2>&1
  ncu -i /tmp/full_$K.ncu-rep --page raw --csv > $O/ncu_vote_L256_${K}_raw.csv 2>/dev/null
done
for L in 32 64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o /tmp/fullL$L python tools/profile_vote.py --levels $L --kinds noise --reps 1 > $O/ncu_full_L$L.log 2>&1
  python tools/ncu_summary.py /tmp/fullL$L.ncu-rep > $O/ncu_vote_L${L}_noise.txt 2>&1
done
bash tools/synth_gpu.sh 2>/dev/null; cp -r gpurun_out/synth $O/ 2>/dev/null
for L in 256 128 64 32 16 8; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > $O/kernel_L$L.json 2>&1; done
