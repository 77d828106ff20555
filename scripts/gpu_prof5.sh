mkdir -p gpurun_out
CMD="python scripts/sweep.py --kf 6 --rows 0 --iters 60 --reps 1"
$CMD > gpurun_out/plain_sweep_6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 10 -c 1 -o gpurun_out/prof_v5_kf6 $CMD > gpurun_out/ncu_v5_6.log 2>&1
tail -1 gpurun_out/ncu_v5_6.log; ls -la gpurun_out
