mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_items.log 2>&1; tail -3 gpurun_out/pytest_items.log
for c in C2 C4; do timeout 500 python scripts/restrict_sweep.py --config $c --reps 3; done > gpurun_out/restrict_items.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_items.json 2> gpurun_out/bench_items.err
