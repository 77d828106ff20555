# Two-phase form of the grouped kernel (RDS_GRP_2PH=1) against the one-phase form: compact tests
# with it on, then the split A/B at C3 / C2 with each.
T=r02s2g
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
RDS_GRP_2PH=1 timeout 900 python -m pytest tests/test_gpu_compact.py -q > gpurun_out/${T}_pytest_compact_2ph.log 2>&1
tail -3 gpurun_out/${T}_pytest_compact_2ph.log
for v in 0 1; do
  RDS_GRP_2PH=$v timeout 600 python scripts/split_ab.py --config C3 > gpurun_out/${T}_split_c3_2ph$v.jsonl 2> gpurun_out/${T}_split_c3_2ph$v.err
  RDS_GRP_2PH=$v timeout 300 python scripts/split_ab.py --config C2 --deltas 0.02 > gpurun_out/${T}_split_c2_2ph$v.jsonl 2> gpurun_out/${T}_split_c2_2ph$v.err
  echo "2PH=$v"; cat gpurun_out/${T}_split_c3_2ph$v.jsonl gpurun_out/${T}_split_c2_2ph$v.jsonl | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['delta_rel'], 'grouped', round(d['grouped_loop_ms'],3), '+setup', round(d['grouped_setup_ms'],3), 'barrier_px', d['barrier_px'], d['same_u'])"
done
