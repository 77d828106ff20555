# Compact path with neighbour synchronisation (k_rdc_iter NB) vs the grid barrier: compact tests,
# then an alternating A/B of the compact K-loop on C3, C2, C1.
mkdir -p gpurun_out
OUT=gpurun_out/r02be_ab.log
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02be_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_compact.py -q -x > gpurun_out/r02be_pytest.log 2>&1
tail -2 gpurun_out/r02be_pytest.log >> $OUT
for rep in 1 2; do for nb in 0 1; do
  echo "== NB=$nb rep=$rep" >> $OUT
  for c in C3 C2 C1; do
  RDS_RDC_NB=$nb timeout 300 python scripts/compact_sweep.py --config $c --deltas 0.02 0.05 0.1 --reps 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$c', d['delta_rel'], round(d['compact_loop_ms'],3), round(d['dense_loop_ms'],3), d.get('same_u'))
" >> $OUT
  done
done; done
cat $OUT
