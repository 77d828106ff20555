# compact path: one-cluster form vs grid-barrier form on small bands (RDS_RDC_CLUSTER=0/1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compact.py -q -x > gpurun_out/cl_pytest.log 2>&1; tail -1 gpurun_out/cl_pytest.log
for c in 1 0; do
  export RDS_RDC_CLUSTER=$c
  timeout 300 python scripts/table1.py --config C0 --qs 0.05,0.2,1 > gpurun_out/cl_t1_$c.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/cl_t1_$c.jsonl'):
    d=json.loads(l)
    if 'q' in d: print('cluster=$c q', d['q'], 'iters', d['iters'], d['compact_iters'], 'dense', round(d['loop_ms'],4), 'compact', round(d['compact_loop_ms'],4))
"
done
