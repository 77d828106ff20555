mkdir -p gpurun_out
for c in C1 C2; do timeout 600 python scripts/restrict_sweep.py --config $c --reps 3; done 2>&1 | tee gpurun_out/restrict1.log
timeout 900 python scripts/restrict_sweep.py --config C4 --reps 2 2>&1 | tee -a gpurun_out/restrict1.log
