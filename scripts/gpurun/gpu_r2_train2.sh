#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train_ops.py tests/test_gpu_train_tenant.py tests/test_gpu_train_step.py tests/test_gpu_dp.py -x -q 2>&1 | tail -4
timeout 300 python scripts/train_trace.py resnet50 64 224 2>&1 | head -12
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 --allreduce > gpurun_out/bench_d4_ar.json 2> gpurun_out/bench_d4_ar.err; head -c 200 gpurun_out/bench_d4_ar.json; echo; tail -c 300 gpurun_out/bench_d4_ar.err
