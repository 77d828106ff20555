mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/r02f_pytest_res.log 2>&1
tail -3 gpurun_out/r02f_pytest_res.log
timeout 300 python scripts/resident_ab.py > gpurun_out/r02f_resident_ab.jsonl 2>&1
cat gpurun_out/r02f_resident_ab.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1
tail -8 gpurun_out/r02f_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02f_pytest.log 2>&1
tail -3 gpurun_out/r02f_pytest.log
