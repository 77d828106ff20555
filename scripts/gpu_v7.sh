# packed-pair (FFMA2) stencil: parity, then a k_fuse sweep at C3 (delta = inf)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest_v7.log; tail -3 gpurun_out/pytest_v7.log
timeout 600 python scripts/sweep.py --kf 4,5,6,7 --rows 0 --reps 3 2>&1 | tee gpurun_out/sweep_v7.log | tail -10
