#!/bin/bash
# quick iteration: GPU tests, k-block timeline, per-op microbench, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/kblock_timeline.py v16_c4 v16_c1_2 r50_l4_exp 2>&1 | grep -v Warn | tail -40
timeout 300 python scripts/op_microbench.py 2>&1 | tail -17 | cut -c1-200
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.err; cut -c1-2500 gpurun_out/bench.json
