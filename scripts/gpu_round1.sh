mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r01_gpu.txt
timeout 1200 python -m pytest tests -m "gpu and not slow" -q 2>&1 | tail -5 > gpurun_out/r01_pytest.log
timeout 600 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$BCMD > gpurun_out/r01_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $BCMD > gpurun_out/r01_ncu_launch.log 2>&1
SCMD="python scripts/sweep.py --kf 5 --rows 0 --iters 60 --reps 1"
$SCMD > gpurun_out/r01_sweep_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 12 -c 1 -o gpurun_out/r01_stencil_kf5 $SCMD > gpurun_out/r01_ncu_full.log 2>&1
ls -la gpurun_out
