# A/B of the rank policy (GACER_RANK_MODE) on the mix, priority partition
for m in 0 3; do echo "RANK_MODE $m"; GACER_RANK_MODE=$m PARTITIONS=priority timeout 300 python scripts/plan_sweep.py 2>&1 | grep -E "identity|split2\"|split4\"|split8" | cut -c1-110; done
GACER_RANK_MODE=3 GACER_PARTITION=priority timeout 300 python scripts/chain_mix.py all_ops_batch_split8 > gpurun_out/chain_mix_r3.txt 2>&1; grep -E "==|totals|mix round" gpurun_out/chain_mix_r3.txt
GACER_RANK_MODE=3 GACER_PARTITION=priority timeout 300 python scripts/busy_analysis.py all_ops_batch_split8 2>&1 | tail -12
