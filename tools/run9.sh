mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/b9_c3.json 2> gpurun_out/b9_c3.err
for wl in c2 c4 c5 c1; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/b9_$wl.json 2> gpurun_out/b9_$wl.err; done
for wl in c3 c4 c5; do TFG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload $wl --steps 5 --warmup 3 > gpurun_out/b9_gloo2_$wl.json 2> gpurun_out/b9_gloo2_$wl.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glcm -s 96 -c 24 --csv --log-file gpurun_out/launches9.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu9.log 2>&1
