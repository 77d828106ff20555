mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ai_build.log 2>&1
for mb in 1 2 3 4; do for npt in 2 8 16; do
  echo "== MAXB=$mb MAXNPT=$npt"
  RDS_RDC_MAXB=$mb RDS_RDC_MAXNPT=$npt timeout 300 python scripts/compact_sweep.py --config C3 --deltas 0.05 0.1 --reps 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['delta_rel'], round(d['compact_loop_ms'],2))
"
done; done
