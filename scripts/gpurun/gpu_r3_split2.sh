#!/bin/bash
# split-K for conv vs swap-AB linears, with / without wider M-pairs; D2, D3, Table-2 mixes (identity plan)
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |"; }
for rep in 1 2; do
  run X=1
  run GACER_SPLITK_MAX=1
  run GACER_SPLITK_MAX=1 GACER_SPLITK_SWAP_MAX=1
  run GACER_SPLITK_MAX=1 GACER_MPAIR_CIN_MAX=4096
  run GACER_SPLITK_MAX=2 GACER_MPAIR_CIN_MAX=4096
done
for c in d3_five t2_r50_v16_m3 t2_r101_d121_m3 t2_alex_v16_r18; do
  for e in X=1 GACER_SPLITK_MAX=1 "GACER_SPLITK_MAX=1 GACER_SPLITK_SWAP_MAX=1" "GACER_SPLITK_MAX=1 GACER_MPAIR_CIN_MAX=4096"; do run GACER_AB_CONFIG=$c $e; done
done
