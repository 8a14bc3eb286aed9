mkdir -p gpurun_out
for K in smooth; do for L in 256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o /tmp/prof8_${K}_L$L python tools/profile_vote.py --levels $L --kinds $K --reps 1 > gpurun_out/ncu8.log 2>&1
  python tools/ncu_summary.py /tmp/prof8_${K}_L$L.ncu-rep > gpurun_out/sum8_${K}_L$L.txt 2>&1
  ncu -i /tmp/prof8_${K}_L$L.ncu-rep --page source --csv --print-source sass > gpurun_out/src8_${K}_L$L.csv 2>/dev/null
done; done
