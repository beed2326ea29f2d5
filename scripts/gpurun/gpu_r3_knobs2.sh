#!/bin/bash
# tile-shape / claim knobs after the split-K change; D2, D3, R101+D121+M3 (identity plan)
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |"; }
for c in d2_r50_v16_mv2 d3_five t2_r101_d121_m3; do
  for rep in 1 2; do
    for e in X=1 GACER_WIDE_GFLOP=0 GACER_WIDE_GFLOP=0.5 GACER_MPAIR_PER_SM=1 GACER_CLAIM_AHEAD=0 GACER_CC_ITEMS_PER_SM=1; do
      run GACER_AB_CONFIG=$c $e
    done
  done
done
