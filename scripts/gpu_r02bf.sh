# Same-box A/B of the whole bench step: this session's code vs the round-2 state at 9ebe161
# (_ab_old/, a git archive), alternating; then the ncu capture of the headline stencil launch.
mkdir -p gpurun_out
OUT=gpurun_out/r02bf_ab.log
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bf_build.log 2>&1
(cd _ab_old && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/r02bf_build_old.log 2>&1)
for rep in 1 2 3; do
  for tree in . _ab_old; do
    (cd $tree && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import sys, json
b = json.loads(sys.stdin.read())
print('$tree rep=$rep', round(b['value'], 1), b['clocks']['sm_mhz'], round(b['roofline']['frac'], 4),
      [(p['delta_rel'], p['path'], round(p['loop_ms'], 3)) for p in b['per_delta']])
") >> $OUT
  done
done
SCMD="python scripts/sweep.py --kf 7 --rows 0 --iters 70 --reps 1 --ws 0"
$SCMD > gpurun_out/r02bf_sweep_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 12 -c 1 -o gpurun_out/r02bf_stencil_kf7 $SCMD > gpurun_out/r02bf_ncu_full.log 2>&1
cat $OUT
OUT2=gpurun_out/r02bf_nb.log
: > $OUT2
timeout 900 python -m pytest tests/test_gpu_compact.py -q -x > gpurun_out/r02bf_pytest_compact.log 2>&1
tail -1 gpurun_out/r02bf_pytest_compact.log >> $OUT2
for rep in 1 2; do for nb in 0 1; do
  echo "== NB=$nb rep=$rep" >> $OUT2
  for c in C3 C2 C1; do
  RDS_RDC_NB=$nb timeout 300 python scripts/compact_sweep.py --config $c --deltas 0.02 0.05 0.1 --reps 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$c', d['delta_rel'], round(d['compact_loop_ms'],3), round(d['dense_loop_ms'],3), d.get('same_u'))
" >> $OUT2
  done
done; done
cat $OUT2
