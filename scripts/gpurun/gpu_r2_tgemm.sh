#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/train_gemm_bench.py 2>&1 | tail -8
for w in dgrad wgrad; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gacer_executor --csv python scripts/one_train_gemm.py $w > gpurun_out/ncu_train_$w.csv 2>&1; echo "$w rc=$?"
done
