#!/bin/bash
mkdir -p gpurun_out
./scripts/micro/epi_bench 2>&1 | tail -30
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariance.py -q -s -k "rne or d3_full or graph_baselines or occupancy" 2>&1 | grep -E "K=|passed|failed|Error|assert" | tail -30
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python scripts/sanitize_round.py d2 > gpurun_out/sanitizer_memcheck_d2.log 2>&1
echo "memcheck d2 rc=$?"; tail -4 gpurun_out/sanitizer_memcheck_d2.log
