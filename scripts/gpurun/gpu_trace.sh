#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/trace_round.py 2>&1 | tail -3
python - <<'PY'
import json
d=json.load(open('gpurun_out/trace_summary.json'))
print({k:v for k,v in d.items() if k!='ops'})
for o in sorted(d['ops'],key=lambda o:o['op']):
  print('%3d %-13s %5d [%7.1f %7.1f] dur %6.1f mean %6.2f max %6.2f sm %8.1f'%(o['op'],o['tenant'],o['items'],o['start_us'],o['end_us'],o['end_us']-o['start_us'],o['item_us_mean'],o['item_us_max'],o['sm_us']))
PY
