#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (run under gpurun); logs in gpurun_out/sanitizer/
mkdir -p gpurun_out/sanitizer
for tool in ${@:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py \
    > gpurun_out/sanitizer/$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer/$tool.log
done
