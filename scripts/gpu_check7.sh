mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest7.log; tail -2 gpurun_out/pytest7.log
timeout 600 python scripts/sweep.py --kf 6 --rows 0 --reps 3 2>&1 | tee gpurun_out/sweep7.log | tail -40
