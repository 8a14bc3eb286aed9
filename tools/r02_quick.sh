#!/bin/bash
# quick A/B: per-L rates + parity subset. Usage: bash tools/r02_quick.sh TAG "levels..." [pytest -k expr]
O=gpurun_out/q_$1; mkdir -p $O
for L in $2; do
  timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/L$L.json 2>&1
done
if [ -n "$3" ]; then timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$3" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; fi
