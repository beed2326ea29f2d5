#!/bin/bash
# one GPU session: tests, bench, ncu launch list + full capture of the executor
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_round.py --rounds 3 > /dev/null 2>&1; wc -l gpurun_out/launches.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_seq.csv python scripts/profile_round.py --rounds 2 --mode sequential > /dev/null 2>&1; wc -l gpurun_out/launches_seq.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 1 -c 1 -o gpurun_out/prof_exec python scripts/profile_round.py --rounds 2 > gpurun_out/ncu_full.log 2>&1; tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out
