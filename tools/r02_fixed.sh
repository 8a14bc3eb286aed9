#!/bin/bash
O=gpurun_out/fixed; mkdir -p $O
for sz in 1024 2048 4096 8192 16384; do
  for L in 256 128 32; do timeout 300 python tools/profile_vote.py --size $sz --levels $L --dts 1:0 --reps 9 --time > $O/s${sz}_L$L.json 2>&1; done
done
# where the fixed cost goes: ncu of a 2048^2 L=256 launch
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote -c 1 -f -o $O/small python tools/profile_vote.py --size 2048 --levels 256 --kinds noise --dts 1:0 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/small.ncu-rep --sass 40 > $O/small.txt 2>&1
ncu -i $O/small.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/small.sass.csv.gz; rm -f $O/small.ncu-rep
