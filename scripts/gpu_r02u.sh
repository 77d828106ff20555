mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02u_build.log 2>&1
timeout 300 python scripts/grid_one.py C1
timeout 300 python scripts/grid_one.py 256x1024
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q > gpurun_out/r02u_pytest_grid.log 2>&1
tail -15 gpurun_out/r02u_pytest_grid.log
