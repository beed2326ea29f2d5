#!/bin/bash
for rep in 1 2; do
  GACER_LIB=$PWD/ab_libs/V8.so timeout 300 python scripts/ab_quick.py 2>&1 | tail -1
  GACER_NO_IM2COL8=1 GACER_LIB=$PWD/ab_libs/V8.so timeout 300 python scripts/ab_quick.py 2>&1 | tail -1
done
for c in d3_five; do
  timeout 600 python bench.py --config $c --plan identity --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c i8', d['ms_per_step'])"
  GACER_NO_IM2COL8=1 timeout 600 python bench.py --config $c --plan identity --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c gather', d['ms_per_step'])"
done
