mkdir -p gpurun_out
CMD="python scripts/sweep.py --kf 6 --rows 128 --iters 60 --reps 1"
$CMD > gpurun_out/plain_sweep.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 10 -c 1 -o gpurun_out/prof_stencil_kf6 $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
BCMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$BCMD > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $BCMD > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log; ls -la gpurun_out
