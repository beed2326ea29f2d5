#!/bin/bash
timeout 300 python scripts/kblock_timeline.py v16_c1_2 r50_l4_exp 2>&1 | grep -v Warn | grep "item\|==" | head -40
