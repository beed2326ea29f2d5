#!/bin/bash
# quick GPU check: parity tests only, bounded
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "conv_op or d1 or cuda_core" 2>&1 | tail -30
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
