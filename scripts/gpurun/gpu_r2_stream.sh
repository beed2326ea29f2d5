#!/bin/bash
# staged streaming operators: training tests (bitwise vs the call-by-call trainer), step anatomy, budget test, D4
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_train_tenant.py tests/test_gpu_train_ops.py tests/test_gpu_invariance.py -x -q 2>&1 | tail -5
timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | head -30
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 > gpurun_out/bench_d4.json 2> gpurun_out/bench_d4.err; tail -c 600 gpurun_out/bench_d4.err; cut -c1-1800 gpurun_out/bench_d4.json
