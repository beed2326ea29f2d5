#!/bin/bash
# same-box A/B of an env switch: tenant_alone + bench makespan, alternating twice
VAR=${VAR:-GACER_NO_MPAIR}
for rep in 1 2; do
  for v in "" 1; do
    echo "== $VAR=$v (rep $rep)"
    env $VAR=$v timeout 300 python scripts/tenant_alone.py 2>&1 | tail -5 | cut -c1-60
    env $VAR=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step'],4), d['config']['plan'], 'seq', round(d['baselines']['sequential']['ms_per_round'],4), 'ms', round(d['baselines']['multistream']['ms_per_round'],4))"
  done
done
