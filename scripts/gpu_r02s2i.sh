# Closing check: compact tests, smoke and the default bench on the final tree.
T=r02s2i
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_strips.py -q > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -c 300 gpurun_out/${T}_bench.err
python -c "
import json; b=json.load(open('gpurun_out/${T}_bench.json')); print(b['value'], b['ms_per_step'], b['gpu_launches'], b['roofline']['frac'], b['clocks'], [(p['delta_rel'],p['path'],round(p['loop_ms'],2),round(p['setup_ms'],2)) for p in b['per_delta']])"
