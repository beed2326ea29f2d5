#!/bin/bash
# in-flight depth 2 for an op's last #CTAs items (GACER_TAIL_DEPTH), same-box A/B
for rep in 1 2; do
  for lib in default tailcc; do
    if [ $lib = default ]; then unset GACER_LIB; else export GACER_LIB=$PWD/ab_libs/tailcc.so; fi
    timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$lib d2] |"
    GACER_AB_CONFIG=d3_five timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$lib d3] |"
    GACER_AB_CONFIG=t2_r101_d121_m3 timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$lib t2r101] |"
    GACER_AB_MIX=vgg16:64 timeout 300 python scripts/ab_mix.py 2>&1 | tail -1 | sed "s|^|[$lib v16@64] |"
  done
done
