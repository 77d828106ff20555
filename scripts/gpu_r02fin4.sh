# Last check of the round on the final commit: the whole GPU test suite, smoke, the default bench
# and the reference arm (no profiler).
T=r02fin4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
python -c "
import json; b=json.load(open('gpurun_out/${T}_bench.json')); print(b['value'], b['ms_per_step'], b['gpu_launches'], b['roofline']['frac'], b['e2e']['value'], b['clocks'])
r=json.load(open('gpurun_out/${T}_ref.json')); print('ref', r['value'])"
