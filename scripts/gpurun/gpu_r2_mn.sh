#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train_ops.py -x -q -k "wgrad" 2>&1 | tail -15
timeout 1200 python -m pytest tests/test_gpu_train_tenant.py tests/test_gpu_train_step.py -x -q 2>&1 | tail -5
timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | head -24
