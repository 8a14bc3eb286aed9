mkdir -p gpurun_out
for wl in c3 c2 c4 c1 c5; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench5_$wl.json 2> gpurun_out/bench5_$wl.err; done
for wl in c2 c4; do timeout 600 python bench.py --impl reference --workload $wl --steps 3 --warmup 3 > gpurun_out/bench5_ref_$wl.json 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tfg:: -s 192 -c 48 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 2 -o gpurun_out/prof_L32 python tools/profile_vote.py --levels 32 --kinds noise,smooth --reps 1 > gpurun_out/ncu_L32.log 2>&1
