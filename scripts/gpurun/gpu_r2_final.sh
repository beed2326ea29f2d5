#!/bin/bash
# round-2 measurement set: bench lines (D2 default = the driver's, D4 plain and with A12, D3, Table-2 mixes),
# launch list of the bench command, ncu full set of the D2 executor and of the D4 training executor round
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 > gpurun_out/bench_d4.json 2> gpurun_out/bench_d4.err; tail -c 300 gpurun_out/bench_d4.err
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 --allreduce > gpurun_out/bench_d4_ar.json 2> gpurun_out/bench_d4_ar.err; tail -c 300 gpurun_out/bench_d4_ar.err
for c in d3_five t2_r50_v16_m3 t2_r101_d121_m3 t2_alex_v16_r18 d1_tiny; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-search > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 200 gpurun_out/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --plan identity --no-cpu-baseline > /dev/null 2>&1; echo ncu-launch rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 2 -c 1 -o gpurun_out/prof_exec_d2 python scripts/profile_round.py --rounds 3 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
timeout 300 python scripts/train_trace.py resnet50 64 224 > gpurun_out/train_trace.txt 2>&1; head -25 gpurun_out/train_trace.txt
ls gpurun_out
