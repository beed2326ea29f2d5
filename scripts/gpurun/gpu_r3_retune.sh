#!/bin/bash
# re-tune the window-item size after the split-K / M-pair changes (identity plan)
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |"; }
for c in d2_r50_v16_mv2 d3_five; do
  for rep in 1 2; do
    for e in X=1 GACER_WIN_ITEMS_PER_SM=0.35 GACER_WIN_ITEMS_PER_SM=0.75 GACER_WIN_ITEMS_PER_SM=1; do run GACER_AB_CONFIG=$c $e; done
  done
done
