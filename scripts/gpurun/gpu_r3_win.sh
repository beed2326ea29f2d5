#!/bin/bash
# window-op item sizing on D2 and D3 (identity plan), interleaved
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |"; }
for rep in 1 2; do
  for w in 2 1 0.5 0.25; do run GACER_WIN_ITEMS_PER_SM=$w; done
done
for rep in 1; do
  for w in 2 1 0.5; do run GACER_AB_CONFIG=d3_five GACER_WIN_ITEMS_PER_SM=$w; done
  for w in 2 1 0.5; do run GACER_AB_CONFIG=t2_r101_d121_m3 GACER_WIN_ITEMS_PER_SM=$w; done
done
