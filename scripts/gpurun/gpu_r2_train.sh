#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train_ops.py -x -q 2>&1 | tail -5
timeout 1200 python -m pytest tests/test_gpu_train_tenant.py -x -q -s 2>&1 | tail -30
