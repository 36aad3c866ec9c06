#!/bin/bash
# compute-sanitizer over tools/san_case.py; logs to gpurun_out/san_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in single loopback; do
    timeout 900 $CS --tool $tool \
      --print-limit 50 python tools/san_case.py $case > gpurun_out/san_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" >> gpurun_out/san_summary.txt
    tail -3 gpurun_out/san_${tool}_${case}.log >> gpurun_out/san_summary.txt
  done
done
