#!/bin/bash
# Round-2 evidence pass (run under gpurun). Outputs in gpurun_out/r02e/ (profiles/README.md).
O=${R02_OUT:-gpurun_out/r02e}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/info.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for b in dropin_tests refsuite_unit refsuite_accept; do timeout 900 tests/cpp/_build/$b > $O/cpp_$b.log 2>&1; echo "rc=$?" >> $O/cpp_$b.log; done
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --impl reference > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
for wl in c2 c4 c5 c1; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 > $O/bench_$wl.json 2> $O/bench_$wl.err; done
# one timed c3 step's launch list (8 launches: 4 KSEL groups x 2 images; cold, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glcm -s 32 -c 8 --csv --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
# ncu --set full of the dominant kernels: L=256 (c3) noise/smooth, L=64 (c5), L=32 (c4), the c2 jobs launch
cap() { # name, profile_vote args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:glcm_vote -c 1 -f -o $O/$1 python tools/profile_vote.py ${@:2} --reps 1 > $O/$1.log 2>&1
  python tools/ncu_summary.py $O/$1.ncu-rep --sass 30 > $O/$1.txt 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/$1.raw.csv.gz
  rm -f $O/$1.ncu-rep
}
cap vote_L256_noise --levels 256 --kinds noise --dts 1:0
cap vote_L256_smooth --levels 256 --kinds smooth --dts 1:0
cap vote_L64_noise_c5 --levels 64 --kinds noise --dts 1:0 --size 16384
cap vote_L32_noise --levels 32 --kinds noise --dts 1:0
cap jobs_c2_L32_noise --levels 32 --kinds noise --dts 1:0,1:45,1:90,1:135 --size 4096 --multi
cap jobs1_c3_L256_noise --levels 256 --kinds noise --dts 1:90,2:90,4:90 --multi
cap jobs1_c3_L256_smooth --levels 256 --kinds smooth --dts 1:90,2:90,4:90 --multi
cap jobs2_c3_L256_noise --levels 256 --kinds noise --dts 1:0,2:0,4:0 --multi
# K0 (Scheme 1, one global atomic per pair) ablation: the paper's contention trend
for L in 8 32 256; do for K in noise smooth; do
  timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,lts__average_t_sector_hit_rate_realtime.pct,l1tex__t_set_conflicts_pipe_lsu_mem_global_op_red.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:glcm_vote_global -c 1 --csv python tools/profile_vote.py --levels $L --kinds $K --dts 1:0 --size 4096 --scheme1 --reps 1 > $O/k0_L${L}_$K.csv 2>&1
  timeout 300 python tools/profile_vote.py --levels $L --kinds $K --dts 1:0 --size 4096 --scheme1 --reps 5 --time > $O/k0_time_L${L}_$K.json 2>&1
  timeout 300 python tools/profile_vote.py --levels $L --kinds $K --dts 1:0 --size 4096 --reps 5 --time > $O/k1_time_L${L}_$K.json 2>&1
done; done
for L in 256 128 64 32 16 8; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > $O/kernel_L$L.json 2>&1; done
bash tools/sanitize.sh > /dev/null 2>&1; cp -r gpurun_out/sanitizer $O/ 2>/dev/null
# per-workload DRAM traffic of one bench step (roofline.traffic)
for wl in c2 c4 c5 c1; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glcm --csv --log-file $O/launches_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/traffic_$wl.log 2>&1
done
timeout 600 ./tools/atomics_bench > $O/atomics.json 2>&1
