mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest3.log; tail -15 gpurun_out/pytest3.log
timeout 600 python scripts/sweep.py --kf 3,4,5,6,7 --rows 0,64,80,96,128 2>&1 | tee gpurun_out/sweep3.log | tail -40
