#!/bin/bash
# full GPU validation + bench lines (D2 default, D4 with the gradient exchange, Table 2 mixes, D3)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.err; cut -c1-600 gpurun_out/bench.json
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 --allreduce > gpurun_out/bench_d4_ar.json 2> gpurun_out/bench_d4_ar.err; tail -c 400 gpurun_out/bench_d4_ar.err; cut -c1-400 gpurun_out/bench_d4_ar.json
timeout 900 python bench.py --config d4_mixed --steps 10 --warmup 3 > gpurun_out/bench_d4.json 2> gpurun_out/bench_d4.err; tail -c 400 gpurun_out/bench_d4.err; cut -c1-400 gpurun_out/bench_d4.json
for c in t2_r50_v16_m3 t2_r101_d121_m3 t2_alex_v16_r18 d3_five; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-search > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.err; cut -c1-300 gpurun_out/bench_$c.json
done
