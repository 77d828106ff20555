mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest5.log; tail -4 gpurun_out/pytest5.log
timeout 600 python scripts/sweep.py --kf 5,6,7 --rows 0,128 2>&1 | tee gpurun_out/sweep5.log | tail -40
for c in C1 C2; do timeout 600 python scripts/restrict_sweep.py --config $c --reps 3; done 2>&1 | tee gpurun_out/restrict5.log
timeout 900 python scripts/restrict_sweep.py --config C4 --reps 2 2>&1 | tee -a gpurun_out/restrict5.log
