# Round 2 evidence: GPU tests (incl. slow), smoke, default bench, the reference arm, ncu launch
# list of a short bench, ncu --set full of the top stencil launch, the resident-cluster kernel,
# the compact kernel at C3 delta = .1 (the headline sweep's compact leg) and the energy kernel.
T=${TAG:-r02p}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-compact"
$BCMD > gpurun_out/${T}_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $BCMD > gpurun_out/${T}_ncu_launch.log 2>&1
SCMD="python scripts/sweep.py --kf 7 --rows 0 --iters 70 --reps 1"
$SCMD > gpurun_out/${T}_sweep_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 12 -c 1 -o gpurun_out/${T}_stencil_kf7 $SCMD > gpurun_out/${T}_ncu_full.log 2>&1
RCMD="python scripts/small_one.py"
$RCMD > gpurun_out/${T}_small_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -s 1 -c 1 -o gpurun_out/${T}_small $RCMD > gpurun_out/${T}_ncu_small.log 2>&1
CCMD="python scripts/compact_one.py --delta-rel 0.1 --iters 30 --split 0"
$CCMD > gpurun_out/${T}_compact_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rdc_iter -c 1 -o gpurun_out/${T}_rdc_iter $CCMD > gpurun_out/${T}_ncu_rdc.log 2>&1
ECMD="python scripts/energy_time.py C3"
$ECMD > gpurun_out/${T}_energy_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_energy_strip -s 2 -c 1 -o gpurun_out/${T}_energy $ECMD > gpurun_out/${T}_ncu_energy.log 2>&1
ls gpurun_out | grep ${T}
