#!/bin/bash
# large-batch mixes (D6(i) Table 3, D5 points 6/7) under the late granularity knobs
run() { env "$@" timeout 300 python scripts/ab_mix.py 2>&1 | tail -1 | sed "s|^|[$*] |"; }
for m in "vgg16:32,resnet18:32" "vgg16:64,mobilenet_v2:64"; do
  for e in X=1 GACER_MPAIR_PER_SM=2 GACER_WIN_ITEMS_PER_SM=2 GACER_CC_ITEMS_PER_SM=1e9 GACER_SPLITK_MAX=4 "GACER_MPAIR_CIN_MAX=64"; do
    run GACER_AB_MIX=$m $e
  done
done
