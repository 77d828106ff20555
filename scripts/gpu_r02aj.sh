mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02aj_build.log 2>&1
for mb in 2 3; do
  echo "== MAXB=$mb"
  for c in C3 C2 C1; do
  RDS_RDC_MAXB=$mb timeout 300 python scripts/compact_sweep.py --config $c --deltas 0.02 0.05 0.1 --reps 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$c', d['delta_rel'], round(d['compact_loop_ms'],3))
"
  done
done
