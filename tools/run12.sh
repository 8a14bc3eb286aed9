mkdir -p gpurun_out
for L in 32 64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o /tmp/prof12_L$L python tools/profile_vote.py --levels $L --kinds noise --reps 1 > gpurun_out/ncu12_L$L.log 2>&1
  python tools/ncu_summary.py /tmp/prof12_L$L.ncu-rep > gpurun_out/sum12_L$L.txt 2>&1
  ncu -i /tmp/prof12_L$L.ncu-rep --page source --csv --print-source sass > gpurun_out/src12_L$L.csv 2>/dev/null
done
