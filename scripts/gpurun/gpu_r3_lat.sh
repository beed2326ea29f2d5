#!/bin/bash
# latency anatomy of the latency-bound tenants + the GPU suite
timeout 300 python scripts/chain_latency.py 2 > gpurun_out/lat_mv2.txt 2>&1; head -40 gpurun_out/lat_mv2.txt
timeout 300 python scripts/chain_latency.py 0 > gpurun_out/lat_r50.txt 2>&1; head -5 gpurun_out/lat_r50.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
