mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest6.log
for L in 256 32 64 128 16 8; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > gpurun_out/t6_L$L.json 2>&1; done
