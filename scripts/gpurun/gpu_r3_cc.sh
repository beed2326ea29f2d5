#!/bin/bash
# per-pixel CC item sizing on the MobileNetV3 / DenseNet mixes; new window default on D2; new-op depth 2
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |; s|$PWD/ab_libs/||"; }
for rep in 1 2; do
  run GACER_WIN_ITEMS_PER_SM=2
  run GACER_WIN_ITEMS_PER_SM=0.5
  run GACER_LIB=$PWD/ab_libs/nd2.so
  for c in 1e9 1 0.5; do run GACER_AB_CONFIG=t2_r50_v16_m3 GACER_CC_ITEMS_PER_SM=$c; done
  for c in 1e9 0.5; do run GACER_AB_CONFIG=t2_r101_d121_m3 GACER_CC_ITEMS_PER_SM=$c; done
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
