import json, sys
t = open(sys.argv[1]).read()
for line in t.splitlines():
    if line.startswith('{"name"'):
        r = json.loads(line)
        print(f"{r['name']:12s} exec {r['executor_us']:7.1f} seq {r['sequential_us']:7.1f} us  exec {r['executor_tflops']:6.1f} TF {r['executor_gbs']:6.0f} GB/s")
    elif line.startswith('{"metric"'):
        r = json.loads(line)
        print("BENCH exec ms %.3f seq %.3f ms %.3f value %.0f e2e %.0f" % (r['ms_per_step'], r['baselines']['sequential']['ms_per_round'],
              r['baselines']['multistream']['ms_per_round'], r['value'], r['e2e']['value']))
    elif line.startswith('op ') or 'sm_busy' in line or 'passed' in line or 'failed' in line or 'Error' in line:
        print(line)
