#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dp.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_train_tenant.py -x -q 2>&1 | tail -3
timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | head -3
