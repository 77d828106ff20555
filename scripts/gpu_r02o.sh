mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -q -k "resident or c0 or ragged or tol" > gpurun_out/r02o_pytest.log 2>&1
tail -3 gpurun_out/r02o_pytest.log
timeout 300 python scripts/resident_ab.py > gpurun_out/r02o_paths.jsonl 2>&1
cat gpurun_out/r02o_paths.jsonl | head -4
timeout 300 python scripts/sweep.py --kf 7 --rows 96,112,128,144,160 --reps 3 > gpurun_out/r02o_rows.jsonl 2>&1
cat gpurun_out/r02o_rows.jsonl
