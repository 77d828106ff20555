# ncu full capture of the packed-pair stencil (KF=6, C3, delta=inf)
mkdir -p gpurun_out
SCMD="python scripts/sweep.py --kf 6 --rows 0 --iters 60 --reps 1"
$SCMD > gpurun_out/prof_v7_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 12 -c 1 -o gpurun_out/prof_v7_kf6 $SCMD > gpurun_out/prof_v7_ncu.log 2>&1
tail -3 gpurun_out/prof_v7_ncu.log
