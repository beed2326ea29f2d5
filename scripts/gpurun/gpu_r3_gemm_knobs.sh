#!/bin/bash
# GEMM item knobs on D2 / D3 (identity plan), interleaved
run() { env "$@" timeout 300 python scripts/ab_d2.py 2>&1 | tail -1 | sed "s|^|[$*] |"; }
for rep in 1 2; do
  run X=1
  run GACER_MPAIR_CIN_MAX=4096
  run GACER_SPLITK_MAX=2
  run GACER_SPLITK_MAX=1
done
for e in X=1 GACER_SPLITK_MAX=2 GACER_SPLITK_MAX=1; do run GACER_AB_CONFIG=d3_five $e; done
