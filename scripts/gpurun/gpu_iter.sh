#!/bin/bash
# one iteration: GPU tests, microbench, bench, trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/op_microbench.py 2>&1 | tail -14
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.err; cut -c1-2500 gpurun_out/bench.json
timeout 300 python scripts/trace_round.py 2>&1 | tail -32
