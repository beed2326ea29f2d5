#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for cfg in next2 d4s; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_round.py $cfg > gpurun_out/sanitizer_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$?"; tail -2 gpurun_out/sanitizer_${tool}_${cfg}.log
  done
done
