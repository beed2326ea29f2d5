#!/bin/bash
# ncu --set full of single-op rounds (executor kernel) for a few characteristic layers
mkdir -p gpurun_out
for op in ${OPS:-v16_c1_2 v16_c4 r50_l4_exp}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 3 -c 1 \
    -o gpurun_out/prof_$op python scripts/op_microbench.py --only $op --reps 3 > gpurun_out/ncu_$op.log 2>&1
  tail -1 gpurun_out/ncu_$op.log
done
