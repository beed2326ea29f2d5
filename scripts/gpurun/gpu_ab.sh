#!/bin/bash
for rep in 1 2; do
for lib in ab_libs/r1.so ab_libs/epi0.so ab_libs/epi1.so; do
  GACER_LIB=$PWD/$lib timeout 300 python scripts/ab_d2.py 2>&1 | tail -1
done
GACER_NO_STATS=1 GACER_LIB=$PWD/ab_libs/epi0.so timeout 300 python scripts/ab_d2.py 2>&1 | tail -1
done
