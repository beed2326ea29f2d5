#!/bin/bash
# bench + ncu evidence for profiles/ (launch list of the bench command; full capture of the executor)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 800 gpurun_out/bench.err; cut -c1-3000 gpurun_out/bench.json
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
CPID=$!
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --plan identity --no-cpu-baseline > /dev/null 2>&1
kill $CPID
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 2 -c 1 -o gpurun_out/prof_exec_d2 python scripts/profile_round.py --rounds 3 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
ls -la gpurun_out
