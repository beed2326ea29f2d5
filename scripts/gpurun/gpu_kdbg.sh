#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/kblock_timeline.py 2>&1 | tail -80
echo "=== AROWS 1x1"
GACER_AROWS_1X1=1 timeout 300 python scripts/kblock_timeline.py r50_l4_exp big_1x1 2>&1 | tail -30
GACER_AROWS_1X1=1 timeout 300 python scripts/op_microbench.py --only _exp 2>&1 | tail -4
timeout 300 python scripts/op_microbench.py --only _exp 2>&1 | tail -4
