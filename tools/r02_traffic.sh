#!/bin/bash
# ncu launch lists (time + DRAM bytes) of one bench step per workload: roofline.traffic
O=gpurun_out/traffic; mkdir -p $O
for wl in c2 c4 c5 c1; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glcm --csv --log-file $O/launches_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$wl.log 2>&1
done
