mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02i_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_resident.py tests/test_gpu_persist.py tests/test_gpu_strips.py -x -q > gpurun_out/r02i_pytest_new.log 2>&1
tail -3 gpurun_out/r02i_pytest_new.log
timeout 600 python scripts/resident_ab.py > gpurun_out/r02i_paths.jsonl 2>&1
cat gpurun_out/r02i_paths.jsonl
