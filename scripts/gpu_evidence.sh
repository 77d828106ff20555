# Round 1 evidence for stencil v7 (FFMA2, KF=7, PDL launches) + f3 compact path: GPU tests (incl. slow), smoke, bench,
# launch list, ncu full capture of the top kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/r01m_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01m_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r01m_bench.json 2> gpurun_out/r01m_bench.err
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-compact"
$BCMD > gpurun_out/r01m_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01m_launches.csv $BCMD > gpurun_out/r01m_ncu_launch.log 2>&1
SCMD="python scripts/sweep.py --kf 7 --rows 0 --iters 70 --reps 1"
$SCMD > gpurun_out/r01m_sweep_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 12 -c 1 -o gpurun_out/r01m_stencil_kf7 $SCMD > gpurun_out/r01m_ncu_full.log 2>&1
tail -2 gpurun_out/r01m_pytest.log; cat gpurun_out/r01m_smoke.log; ls gpurun_out | grep r01m
# f3: the compact kernel (C3 delta = .05, 30 iterations) -- after its own plain run
CCMD="python scripts/compact_one.py --delta-rel 0.05 --iters 30"
$CCMD > gpurun_out/r01m_compact_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rdc_iter -c 1 -o gpurun_out/r01m_rdc_iter $CCMD > gpurun_out/r01m_ncu_rdc.log 2>&1
