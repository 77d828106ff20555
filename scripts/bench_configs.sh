# bench.py on every BASELINE config (C0-C4), one JSON line each -> gpurun_out/bench_configs.jsonl
mkdir -p gpurun_out
: > gpurun_out/bench_configs.jsonl
for c in C0 C1 C2 C3 C4; do
  steps=3; [ $c = C4 ] && steps=1
  timeout 900 python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_configs.jsonl 2> gpurun_out/bench_$c.err
done
python -c "
import json
for l in open('gpurun_out/bench_configs.jsonl'):
    d=json.loads(l); rc=d.get('restricted_compact') or {}
    print(d['config']['workload'][:3], round(d['value'],1), 'roofline', round(d['roofline']['frac'],3), 'MHz', d['clocks']['sm_mhz'],
          [(p['delta_rel'], p['path'], round(p['speedup_vs_full'],2)) for p in rc.get('per_delta', [])])
"
