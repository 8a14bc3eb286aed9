#!/bin/bash
# ncu --set full captures of single vote launches (under gpurun).
# Usage: bash tools/ncu_capture.sh TAG "L:kind:d:theta[:strategy]" ...
# Summaries land in gpurun_out/ncu_TAG_*.txt (+ gzipped raw/source CSV pages);
# the .ncu-rep files are deleted (gpurun copies back <= 64 MiB) unless KEEP_REP=1.
tag=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r L kind d th strat <<< "$spec"
  strat=${strat:-0}
  out=gpurun_out/ncu_${tag}_L${L}_${kind}_d${d}_t${th}_s${strat}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glcm_vote -c 1 -f -o $out \
    python tools/profile_vote.py --levels $L --kinds $kind --dts $d:$th --reps 1 --strategy $strat > $out.log 2>&1
  python tools/ncu_summary.py $out.ncu-rep --sass 30 > $out.txt 2>&1
  ncu -i $out.ncu-rep --page raw --csv 2>/dev/null | gzip > $out.raw.csv.gz
  ncu -i $out.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $out.sass.csv.gz
  [ "${KEEP_REP:-0}" = 1 ] || rm -f $out.ncu-rep
done
