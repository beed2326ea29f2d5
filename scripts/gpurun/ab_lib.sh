#!/bin/bash
# same-box A/B of library builds: default vs $ALT (.so path), alternating twice
ALT=${ALT:-ab_libs/s3db.so}
for rep in 1 2; do
  for lib in "" "$PWD/$ALT"; do
    echo "== lib=${lib:-default} (rep $rep)"
    GACER_LIB=$lib timeout 120 python scripts/tenant_alone.py 2>&1 | tail -5 | cut -c1-60
    GACER_LIB=$lib timeout 240 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step'],4), d['config']['plan'], 'seq', round(d['baselines']['sequential']['ms_per_round'],4), 'ms', round(d['baselines']['multistream']['ms_per_round'],4))"
  done
done
