# Final round-2 evidence (TAG r02h): the standard evidence script, then bench.py on the other
# configs, the 3-D bench, and a same-box bench A/B against the tree at 9ebe161 (_ab_old/).
T=r02h
TAG=$T bash scripts/gpu_evidence_r02.sh
: > gpurun_out/${T}_bench_configs.jsonl
for c in C0 C1 C2 C4; do
  steps=3; [ $c = C4 ] && steps=1
  timeout 900 python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${T}_bench_configs.jsonl 2> gpurun_out/${T}_bench_$c.err
done
timeout 600 python scripts/bench3d.py > gpurun_out/${T}_bench3d.jsonl 2> gpurun_out/${T}_bench3d.err
(cd _ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
OUT=$PWD/gpurun_out/${T}_ab.log
: > $OUT
for rep in 1 2; do for tree in _ab_old .; do
  (cd $tree && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import sys, json
b = json.loads(sys.stdin.read())
print('$tree rep=$rep', round(b['value'], 1), b['clocks']['sm_mhz'], round(b['roofline']['frac'], 4),
      [(p['delta_rel'], p['path'], round(p['loop_ms'], 3)) for p in b['per_delta']])
") >> $OUT
done; done
cat $OUT
ls gpurun_out | grep $T
