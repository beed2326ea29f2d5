#!/bin/bash
# D5 / D6(i) with the late-round-2 defaults, memcheck + synccheck on D2@B=1 and the NEXT-2 mix, D2 spans
mkdir -p gpurun_out/sw
timeout 1200 python scripts/d5_sweep.py > gpurun_out/sw/d5.log 2>&1; echo d5 rc=$?; cp gpurun_out/d5_sweep.json gpurun_out/sw/ 2>/dev/null
timeout 900 python scripts/d6_table3.py > gpurun_out/sw/d6.log 2>&1; echo d6 rc=$?; cp gpurun_out/d6_table3.json gpurun_out/sw/ 2>/dev/null
for tool in memcheck synccheck; do
  for cfg in d2 next2; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_round.py $cfg > gpurun_out/sw/sanitizer_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$?"; tail -2 gpurun_out/sw/sanitizer_${tool}_${cfg}.log
  done
done
timeout 300 python scripts/op_spans.py 1 > gpurun_out/sw/spans_vgg.txt 2>&1
timeout 300 python scripts/op_spans.py 2 > gpurun_out/sw/spans_mv2.txt 2>&1
