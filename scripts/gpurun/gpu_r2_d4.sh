#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --plan identity > gpurun_out/bench_d2_id.json 2> gpurun_out/bench_d2_id.err; tail -c 600 gpurun_out/bench_d2_id.err; python -c "
import json; d=json.load(open('gpurun_out/bench_d2_id.json')); print('D2 identity', d['ms_per_step'], d['value'], {k: v['ms_per_round'] for k, v in d['baselines'].items()})"
timeout 300 python scripts/d7_overheads.py 2>&1 | grep -E "per_op|T_SW|sequential_per"
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 > gpurun_out/bench_d4.json 2> gpurun_out/bench_d4.err; tail -c 1500 gpurun_out/bench_d4.err; cat gpurun_out/bench_d4.json
