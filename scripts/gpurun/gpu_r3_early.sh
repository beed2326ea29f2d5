#!/bin/bash
# early publish of claimed-ahead items: D2 A/B (identity), chain anatomy, D7, GPU suite
L0=$PWD/ab_libs/noearly.so
for rep in 1 2; do
  GACER_LIB=$L0 timeout 300 python scripts/ab_d2.py 2>&1 | tail -1
  timeout 300 python scripts/ab_d2.py 2>&1 | tail -1
done
timeout 300 python scripts/chain_latency.py 2 > gpurun_out/lat_mv2_early.txt 2>&1; head -12 gpurun_out/lat_mv2_early.txt | cut -c1-200
GACER_LIB=$L0 timeout 300 python scripts/d7_overheads.py 2>&1 | grep per_op | sed 's/^/noearly /'
timeout 300 python scripts/d7_overheads.py 2>&1 | grep per_op | sed 's/^/early /'
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
