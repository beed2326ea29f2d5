#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python scripts/d5_sweep.py > gpurun_out/d5.log 2>&1; tail -3 gpurun_out/d5.log | cut -c1-300
timeout 900 python scripts/d6_table3.py > gpurun_out/d6t3.log 2>&1; tail -3 gpurun_out/d6t3.log | cut -c1-300
ls gpurun_out
