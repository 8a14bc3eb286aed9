mkdir -p gpurun_out
for L in 32 256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote_kernel -c 1 -o /tmp/prof7_L$L python tools/profile_vote.py --levels $L --kinds noise --reps 1 > gpurun_out/ncu7_L$L.log 2>&1
  python tools/ncu_summary.py /tmp/prof7_L$L.ncu-rep > gpurun_out/sum7_L$L.txt 2>&1
  ncu -i /tmp/prof7_L$L.ncu-rep --page source --csv --print-source sass > gpurun_out/src7_L$L.csv 2>/dev/null
  ncu -i /tmp/prof7_L$L.ncu-rep --page raw --csv > gpurun_out/raw7_L$L.csv 2>/dev/null
done
