# Round 2, call b: first run of the temporal wavefront (k_wave): bitwise A/B tests, K-loop
# timing A/B per k_fuse and config, then the full GPU suite and the bench with the new default.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_wave.py -x -q > gpurun_out/r02b_pytest_wave.log 2>&1
tail -3 gpurun_out/r02b_pytest_wave.log
timeout 300 python scripts/wave_ab.py --config C3 --kf 4,5,6,7 --check --reps 3 > gpurun_out/r02b_wave_c3.jsonl 2>&1
cat gpurun_out/r02b_wave_c3.jsonl
timeout 300 python scripts/wave_ab.py --config C2 --kf 6 --deltas inf,0.2,0.05 --reps 3 > gpurun_out/r02b_wave_c2.jsonl 2>&1
timeout 300 python scripts/wave_ab.py --config C1 --kf 4,6 --deltas inf,0.2 --reps 3 > gpurun_out/r02b_wave_c1.jsonl 2>&1
timeout 600 python scripts/wave_ab.py --config C4 --kf 6 --deltas inf,0.2 --reps 2 > gpurun_out/r02b_wave_c4.jsonl 2>&1
cat gpurun_out/r02b_wave_c2.jsonl gpurun_out/r02b_wave_c1.jsonl gpurun_out/r02b_wave_c4.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02b_pytest.log 2>&1
tail -3 gpurun_out/r02b_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
