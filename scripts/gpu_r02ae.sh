mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ae_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_vol.py -x -q > gpurun_out/r02ae_pytest_vol.log 2>&1
tail -5 gpurun_out/r02ae_pytest_vol.log
timeout 600 python scripts/bench3d.py --kf 1,2,3 > gpurun_out/r02ae_bench3d.jsonl 2>&1; cat gpurun_out/r02ae_bench3d.jsonl
