#!/bin/bash
# bench.py lines under env A/B: bash tools/r02_benchab.sh TAG "c2 c4" "ENV=0" "ENV=1"
O=gpurun_out/bab_$1; mkdir -p $O
for wl in $2; do
  for e in "${@:3}"; do
    env $e timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 > $O/${wl}_${e//=/_}.json 2> $O/${wl}_${e//=/_}.err
  done
done
