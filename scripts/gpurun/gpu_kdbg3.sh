#!/bin/bash
for sp in 0 1; do echo "spin $sp"; GACER_DBG_SPIN=$sp timeout 300 python scripts/kblock_timeline.py r50_l4_exp v16_c1_2 2>&1 | grep -v Warn | grep "item [0-2]\|==" | head -12; done
