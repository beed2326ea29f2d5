#!/bin/bash
# a large op's first item joining one item in flight (GACER_BIGOP_DEPTH2), same-box A/B
L=$PWD/ab_libs/big2.so
for rep in 1 2; do
  for lib in default big2; do
    if [ $lib = default ]; then unset GACER_LIB; else export GACER_LIB=$L; fi
    timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$lib d2] |"
    GACER_AB_CONFIG=d3_five timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$lib d3] |"
    GACER_AB_MIX=vgg16:64,mobilenet_v2:64 timeout 300 python scripts/ab_mix.py 2>&1 | tail -1 | sed "s|^|[$lib v16+mv2@64] |"
  done
done
