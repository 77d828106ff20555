# Round 2, third session: the compact path's coupled / decoupled split (RDS_OPT_RDC_SPLIT).
T=r02s2a
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_compact.py -q -x > gpurun_out/${T}_pytest_compact.log 2>&1
tail -3 gpurun_out/${T}_pytest_compact.log
timeout 600 python scripts/split_ab.py --config C3 > gpurun_out/${T}_split_c3.jsonl 2> gpurun_out/${T}_split_c3.err
timeout 300 python scripts/split_ab.py --config C2 --deltas 0.02 0.05 0.1 > gpurun_out/${T}_split_c2.jsonl 2> gpurun_out/${T}_split_c2.err
cat gpurun_out/${T}_split_c3.jsonl gpurun_out/${T}_split_c2.jsonl
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -c 600 gpurun_out/${T}_bench.json
