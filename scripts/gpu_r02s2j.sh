# Second-chance trial of the auto mode (scattered bands the barrier model rejects): compact,
# strips and parity tests, then bench.py on C1, C2, C4 and the default C3.
T=r02s2j
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
: > gpurun_out/${T}_bench_configs.jsonl
for c in C1 C2 C4; do
  steps=3; [ $c = C4 ] && steps=1
  timeout 900 python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${T}_bench_configs.jsonl 2> gpurun_out/${T}_bench_$c.err
done
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json
for l in list(open('gpurun_out/${T}_bench_configs.jsonl')) + [open('gpurun_out/${T}_bench.json').read()]:
    c=json.loads(l); print(c['config']['workload'][:3], round(c['value'],1), c['gpu_launches'], [(p['delta_rel'],p['path'],round(p['loop_ms'],3),round(p['setup_ms'],3)) for p in c['per_delta']])"
