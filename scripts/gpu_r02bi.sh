# Stencil-only same-box A/B (sweep.py, C3 K-loop, k_fuse 7, delta inf and .2): the tree at
# 9ebe161 against the current tree with the prologue / edge split / predicated stores on and off.
mkdir -p gpurun_out
OUT=$PWD/gpurun_out/r02bi_ab.log
: > $OUT
(cd _ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
run() {  # tree, defs
  (cd $1 && RDS_NVCC_DEFS="$2" python paper_1807_11534_b200/_build.py > /dev/null 2>&1 || echo "BUILD FAILED $1 [$2]" >> $OUT)
  for dl in inf 0.2; do
    (cd $1 && RDS_NVCC_DEFS="$2" timeout 300 python scripts/sweep.py --kf 7 --rows 0 --delta $dl --reps 7 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print('$1 [$2] delta=$dl', round(d['loop_ms'], 3), d['items'])
") >> $OUT
  done
}
for rep in 1 2 3; do
  run _ab_old ""
  run . ""
  run . "-DRDS_NO_PROLOGUE"
  run . "-DRDS_NO_PROLOGUE -DRDS_EDGE_ALWAYS=1 -DRDS_NO_PRED_STORE"
done
cat $OUT
