mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest2.log; tail -15 gpurun_out/pytest2.log
timeout 600 python scripts/sweep.py --kf 3,4,5,6,7,8 --rows 64,96,128,192,256 2>&1 | tee gpurun_out/sweep2.log | tail -40
