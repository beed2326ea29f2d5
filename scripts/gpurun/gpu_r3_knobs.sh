#!/bin/bash
# item-size knobs on D2 (identity plan), interleaved; env read at registration
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |"; }
for rep in 1 2; do
  run GACER_WIN_ITEMS_PER_SM=2
  run GACER_WIN_ITEMS_PER_SM=1
  run GACER_WIN_ITEMS_PER_SM=4
  run GACER_MPAIR_PER_SM=1
  run GACER_NO_MPAIR=1
  run GACER_WIN_ITEMS_PER_SM=1 GACER_MPAIR_PER_SM=1
done
