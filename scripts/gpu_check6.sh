mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest6.log; tail -2 gpurun_out/pytest6.log
timeout 600 python scripts/sweep.py --kf 4,5,6,7 --rows 0,96,128 2>&1 | tee gpurun_out/sweep6.log | tail -40
for c in C2; do timeout 600 python scripts/restrict_sweep.py --config $c --reps 3; done 2>&1 | tee gpurun_out/restrict6.log | cut -c1-250
