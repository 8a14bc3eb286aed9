#!/bin/bash
O=gpurun_out/p16; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "every_strategy or p16x16 or jobs" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for st in 2 5; do for L in 64 48; do
  timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --strategy $st --time > $O/s${st}_L$L.json 2>&1
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote -c 1 -f -o $O/p16 python tools/profile_vote.py --levels 64 --kinds noise --dts 1:0 --reps 1 --strategy 5 > /dev/null 2>&1
python tools/ncu_summary.py $O/p16.ncu-rep --sass 20 > $O/p16_ncu.txt 2>&1; rm -f $O/*.ncu-rep
