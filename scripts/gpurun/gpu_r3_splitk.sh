#!/bin/bash
# pipelined split-K reduction: D2 A/B (identity) + VGG-16 spans + the GEMM parity tests
L0=$PWD/ab_libs/base.so
for rep in 1 2; do
  GACER_LIB=$L0 timeout 300 python scripts/ab_d2.py 2>&1 | tail -1
  timeout 300 python scripts/ab_d2.py 2>&1 | tail -1
done
timeout 300 python scripts/op_spans.py 1 > gpurun_out/spans_vgg_pipe.txt 2>&1; head -22 gpurun_out/spans_vgg_pipe.txt | cut -c1-150
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
