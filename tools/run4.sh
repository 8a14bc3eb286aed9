mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest4.log
for wl in c3 c2 c4 c1 c5; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench4_$wl.json 2> gpurun_out/bench4_$wl.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench4_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tfg:: -s 192 -c 48 --csv --log-file gpurun_out/launches4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu4.log 2>&1
