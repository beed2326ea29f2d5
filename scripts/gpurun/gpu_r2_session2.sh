#!/bin/bash
# round-2 session-2 baseline: all GPU tests, D2 bench (driver default), D4 bench, launch list + ncu full of the executor
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 800 gpurun_out/bench.err; cut -c1-2500 gpurun_out/bench.json
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 > gpurun_out/bench_d4.json 2> gpurun_out/bench_d4.err; tail -c 800 gpurun_out/bench_d4.err; cut -c1-2500 gpurun_out/bench_d4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --plan identity --no-cpu-baseline > /dev/null 2>&1; echo ncu-launch rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 2 -c 1 -o gpurun_out/prof_exec_d2 python scripts/profile_round.py --rounds 3 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
ls -la gpurun_out
