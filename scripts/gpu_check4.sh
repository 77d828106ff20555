mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest4.log; tail -4 gpurun_out/pytest4.log
timeout 600 python scripts/sweep.py --kf 4,5,6,7 --rows 0,64,128 2>&1 | tee gpurun_out/sweep4.log | tail -40
for kf in 6; do
CMD="python scripts/sweep.py --kf $kf --rows 0 --iters 60 --reps 1"
$CMD > gpurun_out/plain_sweep_$kf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 10 -c 1 -o gpurun_out/prof_v6_kf$kf $CMD > gpurun_out/ncu_v6_$kf.log 2>&1
tail -1 gpurun_out/ncu_v6_$kf.log
done
