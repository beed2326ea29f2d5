#!/bin/bash
# same-box A/B of every ab_libs/*.so: tenants alone/mixed + union-busy analysis
for lib in ab_libs/*.so; do
  echo "=== $lib"
  GACER_LIB=$PWD/$lib timeout 300 python scripts/tenant_alone.py 2>&1 | tail -5
  for p in identity all_ops_batch_split4; do GACER_LIB=$PWD/$lib timeout 300 python scripts/busy_analysis.py $p 2>&1 | grep -E "^plan|union"; done
done
