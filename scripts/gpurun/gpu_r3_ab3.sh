#!/bin/bash
# inline-dependency width x buffer reuse x weight prefetch on D2 (identity plan), interleaved
L8=$PWD/ab_libs/in8.so
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |; s|$PWD/ab_libs/||"; }
for rep in 1 2; do
  run GACER_NO_REUSE=1 GACER_NO_WPREFETCH=1
  run GACER_NO_REUSE=1
  run GACER_NO_REUSE=0
  run GACER_LIB=$L8 GACER_NO_REUSE=1
  run GACER_LIB=$L8 GACER_NO_REUSE=0
  run GACER_LIB=$L8 GACER_REUSE_MIN_KB=4096
done
for v in "GACER_NO_WPREFETCH=1" "GACER_NO_WPREFETCH=0"; do
  env $v timeout 300 python scripts/d7_overheads.py 2>&1 | tail -4 | sed "s/^/[$v] /"
done
