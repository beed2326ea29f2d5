#!/bin/bash
for e in "" "GACER_DGRAD_PHASES=1" "GACER_DGRAD_DILATE=1"; do
  echo "== $e"; env $e timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | head -3
done
timeout 900 python -m pytest tests/test_gpu_train_ops.py -x -q -k "dgrad" 2>&1 | tail -2
