#!/bin/bash
O=gpurun_out/tail; mkdir -p $O
for t in 0 10 25 50; do
  TEXFORGE_POOL_TAIL=$t timeout 300 python tools/profile_vote.py --levels 256 --dts 1:0,1:45,2:90,4:135 --reps 7 --time > $O/t$t.json 2>&1
done
TEXFORGE_POOL_TAIL=25 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "pool or packed16 or appendix_a_c3 or partials or drains" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
