#!/bin/bash
# round-2 baseline: GPU tests, bench, D7 overheads, R50 chain anatomy
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python scripts/d7_overheads.py 2>&1 | tail -15
timeout 300 python scripts/chain_latency.py 0 2>&1 | tail -70
