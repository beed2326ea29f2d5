#!/bin/bash
for ca in 0 1; do
  echo "== GACER_CLAIM_AHEAD=$ca"
  GACER_CLAIM_AHEAD=$ca timeout 300 python scripts/d7_overheads.py 2>&1 | grep -E "per_op|T_SW_dev"
  GACER_CLAIM_AHEAD=$ca timeout 300 python scripts/ab_d2.py 2>&1 | tail -1
  GACER_CLAIM_AHEAD=$ca timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | head -1
done
timeout 1200 python -m pytest tests/test_gpu_invariance.py tests/test_gpu_train_tenant.py -x -q 2>&1 | tail -3
