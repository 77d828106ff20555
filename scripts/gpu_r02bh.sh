# Same-box bench A/B of the stencil changes of this session against the tree at 9ebe161: the
# current tree with each change switched off in turn (RDS_NVCC_DEFS), alternating with the old
# tree.  bench.py rebuilds the library whenever RDS_NVCC_DEFS changes (content hash).
mkdir -p gpurun_out
OUT=$PWD/gpurun_out/r02bh_ab.log
: > $OUT
(cd _ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
run() {  # tree, defs
  (cd $1 && RDS_NVCC_DEFS="$2" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import sys, json
b = json.loads(sys.stdin.read())
print('$1 [$2]', round(b['value'], 1), b['clocks']['sm_mhz'],
      [(p['delta_rel'], round(p['loop_ms'], 3)) for p in b['per_delta']])
") >> $OUT
}
for rep in 1 2; do
  run _ab_old ""
  run . ""
  run . "-DRDS_NO_PRED_STORE"
  run . "-DRDS_NO_PROLOGUE"
  run . "-DRDS_EDGE_ALWAYS=1"
  run . "-DRDS_NO_PRED_STORE -DRDS_NO_PROLOGUE -DRDS_EDGE_ALWAYS=1"
done
cat $OUT
