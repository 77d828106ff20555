# Round 1 (session 2): re-verify HEAD on B200: GPU tests (incl. slow), smoke, bench, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r01c_gpu.txt
nproc > gpurun_out/r01c_nproc.txt; lscpu | grep "Model name" >> gpurun_out/r01c_nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r01c_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01c_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r01c_bench.json 2> gpurun_out/r01c_bench.err
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$BCMD > gpurun_out/r01c_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_launches.csv $BCMD > gpurun_out/r01c_ncu_launch.log 2>&1
ls -la gpurun_out
