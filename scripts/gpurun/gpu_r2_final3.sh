#!/bin/bash
# end-of-round-2 measurement set: GPU suite + smoke, bench lines, D5 / D6(i), launch list, ncu full set, training trace
O=${OUT:-gpurun_out/f5}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; tail -1 $O/gputest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; cut -c1-300 $O/bench.json
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 > $O/bench_d4.json 2> $O/bench_d4.err
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 --allreduce > $O/bench_d4_ar.json 2> $O/bench_d4_ar.err
for c in d3_five t2_r50_v16_m3 t2_r101_d121_m3 t2_alex_v16_r18 d1_tiny; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-search > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python scripts/d7_overheads.py > $O/d7.log 2>&1; cp gpurun_out/d7.json $O/d7.json 2>/dev/null
timeout 1200 python scripts/d5_sweep.py > $O/d5.log 2>&1; cp gpurun_out/d5_sweep.json $O/ 2>/dev/null
timeout 900 python scripts/d6_table3.py > $O/d6.log 2>&1; cp gpurun_out/d6_table3.json $O/ 2>/dev/null
timeout 300 python scripts/train_trace.py resnet50 64 224 > $O/train_trace.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --plan identity --no-cpu-baseline > /dev/null 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gacer_executor -s 2 -c 1 -o $O/prof_exec_d2 python scripts/profile_round.py --rounds 3 > $O/ncu_full.log 2>&1; tail -1 $O/ncu_full.log
ls $O | wc -l
