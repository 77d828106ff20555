# compact-path launch variants (grid cap, register-resident codes) on C3 / C1
mkdir -p gpurun_out
for v in "2 16" "2 2" "4 2" "4 0" "3 2" "1 16"; do
  set -- $v
  export RDS_RDC_MAXB=$1 RDS_RDC_MAXNPT=$2
  for c in C3 C1; do
    timeout 300 python scripts/compact_sweep.py --config $c --deltas 0.02 0.05 0.08 0.1 --reps 3 > gpurun_out/cv_${c}_$1_$2.jsonl 2>&1
    python -c "
import json
for l in open('gpurun_out/cv_${c}_$1_$2.jsonl'):
    d=json.loads(l); print('maxb $1 npt $2', d['config'], d['delta_rel'], 'compact', round(d['compact_loop_ms'],3), 'x', round(d['compact_over_dense'],2), d['same_u'])
"
  done
done
