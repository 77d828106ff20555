# Round 2, fifth session: grouped connected components of the compact path (RDS_OPT_RDC_SPLIT = 2).
T=r02s2f
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_compact.py -q > gpurun_out/${T}_pytest_compact.log 2>&1
tail -5 gpurun_out/${T}_pytest_compact.log
timeout 600 python scripts/split_ab.py --config C3 > gpurun_out/${T}_split_c3.jsonl 2> gpurun_out/${T}_split_c3.err
tail -3 gpurun_out/${T}_split_c3.err
timeout 300 python scripts/split_ab.py --config C2 --deltas 0.02 0.05 0.1 > gpurun_out/${T}_split_c2.jsonl 2> gpurun_out/${T}_split_c2.err
cat gpurun_out/${T}_split_c3.jsonl gpurun_out/${T}_split_c2.jsonl | cut -c1-1400
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -c 300 gpurun_out/${T}_bench.err
python -c "
import json; b=json.load(open('gpurun_out/${T}_bench.json')); print(b['value'], b['ms_per_step'], [(p['delta_rel'],p['path'],round(p['loop_ms'],2),round(p['setup_ms'],2)) for p in b['per_delta']])"
