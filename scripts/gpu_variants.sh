# Compile-time variants of the stencil (RDS_NVCC_DEFS) x launch options, C3 delta = inf.
mkdir -p gpurun_out
OUT=gpurun_out/variants_${TAG:-x}.log
: > $OUT
for defs in ${VARIANTS:-"-DRDS_CHAINS=2"}; do
  d="${defs//,/ } -DRDS_KF_LIST(X)=X(6)X(7)"
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>>$OUT || { echo "build failed: $d" >> $OUT; continue; }
  RDS_NVCC_DEFS="$d" timeout 300 python scripts/sweep.py --kf ${KFS:-6,7} --rows 0 --ctas ${CTAS:-0} --reps 3 >> $OUT 2>&1
done
cat $OUT
