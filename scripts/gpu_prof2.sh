mkdir -p gpurun_out
for kf in 5 6; do
CMD="python scripts/sweep.py --kf $kf --rows 128 --iters 60 --reps 1"
$CMD > gpurun_out/plain_sweep_$kf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 10 -c 1 -o gpurun_out/prof_v3_kf$kf $CMD > gpurun_out/ncu_v3_$kf.log 2>&1
tail -1 gpurun_out/ncu_v3_$kf.log
done
