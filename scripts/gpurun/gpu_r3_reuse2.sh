#!/bin/bash
# reuse / L2-hint variants on D2 (identity plan), interleaved, same box
declare -a V=("GACER_NO_REUSE=1" "GACER_NO_REUSE=0" "GACER_REUSE_MIN_KB=4096" "GACER_REUSE_DIST=3" "GACER_NO_REUSE=1 GACER_NO_L2_HINT=1" "GACER_REUSE_MIN_KB=4096 GACER_REUSE_DIST=3")
for rep in 1 2; do
  for v in "${V[@]}"; do
    env $v timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
done
for v in "GACER_REUSE_MIN_KB=4096" "GACER_NO_REUSE=1 GACER_NO_L2_HINT=1" "GACER_REUSE_DIST=3"; do
  env $v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:gacer_executor -s 1 -c 1 --csv python scripts/profile_round.py --rounds 2 2>&1 | grep -E 'dram__bytes|duration' | awk -F'","' '{print $13, $15}' | sed "s/^/[$v] /"
done
