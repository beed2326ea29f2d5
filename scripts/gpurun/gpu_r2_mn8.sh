#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_train_ops.py -x -q -k "wgrad" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_train_tenant.py tests/test_gpu_train_step.py -x -q 2>&1 | tail -2
timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | head -12
