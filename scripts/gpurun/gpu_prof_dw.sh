#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_cc_kernel -s 2 -c 1 \
  -o gpurun_out/prof_dw python scripts/op_microbench.py --only mv2_dw_s1 --reps 3 > gpurun_out/ncu_dw.log 2>&1
tail -2 gpurun_out/ncu_dw.log
