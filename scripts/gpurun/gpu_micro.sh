#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/op_microbench.py 2>&1 | tail -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 3 -c 1 -o gpurun_out/prof_r50l3 python scripts/op_microbench.py --only r50_l3 --reps 3 > gpurun_out/ncu_r50l3.log 2>&1; tail -2 gpurun_out/ncu_r50l3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 3 -c 1 -o gpurun_out/prof_v16c3 python scripts/op_microbench.py --only v16_c3 --reps 3 > gpurun_out/ncu_v16c3.log 2>&1; tail -2 gpurun_out/ncu_v16c3.log
