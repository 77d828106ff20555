# Occupancy of the grouped compact kernel: k_rdc_grp built with __launch_bounds__(256, m), m = 1
# (60 registers, 4 CTAs per SM), 6, 8 (register caps 40 / 32): split A/B at C3.
T=r02s2h
mkdir -p gpurun_out
OUT=gpurun_out/${T}_grp_minb.txt
: > $OUT
for m in 1 6 8; do
  export RDS_NVCC_DEFS="-DRDS_GRP_MINB=$m"
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build_$m.log 2>&1
  echo "RDS_GRP_MINB=$m" >> $OUT
  cuobjdump -res-usage paper_1807_11534_b200/librds.so 2>/dev/null | grep -A1 "k_rdc_grpE" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | paste - - >> $OUT
  timeout 600 python scripts/split_ab.py --config C3 --deltas 0.02 0.05 0.1 2> gpurun_out/${T}_err_$m.log | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['delta_rel'], 'grouped', round(d['grouped_loop_ms'],3), '+setup', round(d['grouped_setup_ms'],3), 'barrier_px', d['barrier_px'], d['same_u'])" >> $OUT
done
cat $OUT
