# Round 2 closing evidence on the final tree (TAG r02fin): the standard evidence script (GPU tests,
# smoke, bench, reference arm, launch list, ncu captures), an ncu capture of the decoupled-pixel
# kernels k_rdc_iso and k_rdc_grp of the compact path (k_rdc_iter is captured with the split off), then bench.py on the other configs and the 3-D bench.
T=${TAG:-r02fin}
TAG=$T bash scripts/gpu_evidence_r02.sh
CCMD="python scripts/compact_one.py --delta-rel 0.1 --iters 100"
$CCMD > gpurun_out/${T}_compact_grp_plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rdc_iso -c 1 -o gpurun_out/${T}_rdc_iso $CCMD > gpurun_out/${T}_ncu_rdc_iso.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rdc_grp -c 1 -o gpurun_out/${T}_rdc_grp $CCMD > gpurun_out/${T}_ncu_rdc_grp.log 2>&1
: > gpurun_out/${T}_bench_configs.jsonl
for c in C0 C1 C2 C4; do
  steps=3; [ $c = C4 ] && steps=1
  timeout 900 python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${T}_bench_configs.jsonl 2> gpurun_out/${T}_bench_$c.err
done
timeout 600 python scripts/bench3d.py > gpurun_out/${T}_bench3d.jsonl 2> gpurun_out/${T}_bench3d.err
ls gpurun_out | grep $T
