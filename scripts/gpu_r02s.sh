mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02s_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q > gpurun_out/r02s_pytest_grid.log 2>&1
tail -15 gpurun_out/r02s_pytest_grid.log
timeout 300 python scripts/grid_ab.py C1 > gpurun_out/r02s_grid_c1.jsonl 2>&1; cat gpurun_out/r02s_grid_c1.jsonl
timeout 300 python scripts/grid_ab.py 512x512 > gpurun_out/r02s_grid_512.jsonl 2>&1; cat gpurun_out/r02s_grid_512.jsonl
