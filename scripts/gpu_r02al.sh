mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02al_build.log 2>&1
for rep in 1 2; do for mb in 3 2; do
  RDS_RDC_MAXB=$mb timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02al_bench_${mb}_${rep}.json 2>/dev/null
  python -c "
import json
b=json.loads(open('gpurun_out/r02al_bench_${mb}_${rep}.json').read().strip().splitlines()[-1])
print('MAXB=$mb rep=$rep', round(b['value'],1), b['clocks']['sm_mhz'], [(p['delta_rel'],p['path'],round(p['loop_ms'],2)) for p in b['per_delta']])
"
done; done
