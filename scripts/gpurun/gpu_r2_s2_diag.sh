#!/bin/bash
# round-2 session-2 diagnostics: training step anatomy in the executor, D7 overheads, chain latency, sanitizers
mkdir -p gpurun_out
timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | tail -70
timeout 300 python scripts/d7_overheads.py 2>&1 | tail -12; cp gpurun_out/d7.json gpurun_out/d7_s2.json 2>/dev/null
timeout 300 python scripts/chain_latency.py 0 2>&1 | tail -40
for tool in memcheck racecheck synccheck; do
  for cfg in d1 d2; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_round.py $cfg > gpurun_out/sanitizer_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$?"; tail -3 gpurun_out/sanitizer_${tool}_${cfg}.log
  done
done
