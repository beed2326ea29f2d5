#!/bin/bash
# round-2: new parity / invariance / stats / graph-baseline tests, bench with graphed baselines, sanitizers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariance.py -x -q 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_train_step.py -x -q -k "sequential_trainer" 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.err; cat gpurun_out/bench.json
for tool in memcheck racecheck synccheck; do
  for cfg in d1 d2; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_round.py $cfg > gpurun_out/sanitizer_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$?"; tail -4 gpurun_out/sanitizer_${tool}_${cfg}.log
  done
done
