#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2000 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python scripts/trace_round.py 2>&1 | tail -40
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_seq.csv python scripts/profile_round.py --rounds 2 --mode sequential > /dev/null 2>&1
