mkdir -p gpurun_out
timeout 300 python scripts/dbg_timing.py 2>&1 | tail -45
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ncu_small.csv python scripts/op_microbench.py --only r50_l1_1x1 --reps 3 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ncu_small.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['Kernel Name'][:30], d['Metric Name'], d['Metric Value'])
PY
