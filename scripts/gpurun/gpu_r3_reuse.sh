#!/bin/bash
# round 3 (session 3): liveness-based buffer reuse A/B on D2 + DRAM bytes of the executor
mkdir -p gpurun_out
for e in 0 1 0 1; do GACER_NO_REUSE=$e timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s/^/noreuse=$e /"; done
for e in 0 1; do
  GACER_NO_REUSE=$e timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:gacer_executor -s 1 -c 1 --csv python scripts/profile_round.py --rounds 2 > gpurun_out/ncu_dram_noreuse$e.csv 2>&1
  grep -E 'dram__bytes|duration|hit_rate' gpurun_out/ncu_dram_noreuse$e.csv | sed "s/^/noreuse=$e /"
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
GACER_NO_REUSE=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_reuse.json 2> gpurun_out/bench_reuse.err; echo bench rc $?
