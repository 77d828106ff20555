mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ak_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py -x -q -k "compact or tol or c0 or c1" > gpurun_out/r02ak_pytest.log 2>&1
tail -3 gpurun_out/r02ak_pytest.log
timeout 900 python bench.py > gpurun_out/r02ak_bench.json 2> gpurun_out/r02ak_bench.err
python -c "
import json
b=json.loads(open('gpurun_out/r02ak_bench.json').read().strip().splitlines()[-1])
print(b['value'], b['ms_per_step'], b['e2e']['value'], b['roofline']['frac'], b['clocks'])
print([(p['delta_rel'],p['path'],round(p['loop_ms'],2)) for p in b['per_delta']])
"
