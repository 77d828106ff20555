# Compile-time variants of the stencil (RDS_NVCC_DEFS) x launch options, C3 delta = inf.
mkdir -p gpurun_out
OUT=gpurun_out/variants_${TAG:-x}.log
: > $OUT
for defs in ${VARIANTS:-"-DRDS_CHAINS=3"}; do
  d="${defs//,/ } -DRDS_KF_LIST(X)=X(6)X(7)"
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>>$OUT || { echo "build failed: $d" >> $OUT; continue; }
  if [ -n "$PARITY" ]; then RDS_NVCC_DEFS="$d" timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1 or c0 or ragged or fusion" 2>&1 | tail -1 >> $OUT; fi
  RDS_NVCC_DEFS="$d" timeout 300 python scripts/sweep.py --kf ${KFS:-6,7} --rows 0 --ctas ${CTAS:-0} --reps ${REPS:-3} >> $OUT 2>&1
done
cat $OUT
