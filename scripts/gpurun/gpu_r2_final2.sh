#!/bin/bash
# late-round-2 measurement set: GPU suite, bench lines (D2 default = the driver's, D4 plain and with A12,
# D3, Table-2 mixes, D1), launch list of the bench command, ncu full set of the D2 executor, D7
O=${OUT:-gpurun_out/f2}; mkdir -p $O

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.err; cut -c1-400 $O/bench.json
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 > $O/bench_d4.json 2> $O/bench_d4.err; tail -c 200 $O/bench_d4.err
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 --allreduce > $O/bench_d4_ar.json 2> $O/bench_d4_ar.err; tail -c 200 $O/bench_d4_ar.err
for c in d3_five t2_r50_v16_m3 t2_r101_d121_m3 t2_alex_v16_r18 d1_tiny; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-search > $O/bench_$c.json 2> $O/bench_$c.err; tail -c 200 $O/bench_$c.err
done
timeout 300 python scripts/d7_overheads.py > $O/d7.log 2>&1; cp gpurun_out/d7.json $O/d7.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --plan identity --no-cpu-baseline > /dev/null 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 2 -c 1 -o $O/prof_exec_d2 python scripts/profile_round.py --rounds 3 > $O/ncu_full.log 2>&1; tail -2 $O/ncu_full.log
ls $O
