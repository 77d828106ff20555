# Compile-time variants of the temporal wavefront (RDS_NVCC_DEFS), C3 delta = inf, K = 1000:
# K-loop time with and without the wavefront for each k_fuse in $KFS.
mkdir -p gpurun_out
OUT=gpurun_out/wave_variants_${TAG:-x}.log
: > $OUT
for defs in ${VARIANTS:-"-DRDS_WAVE_PUB=4"}; do
  d="${defs//,/ }"
  echo "== $d" >> $OUT
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>>$OUT || { echo "build failed: $d" >> $OUT; continue; }
  RDS_NVCC_DEFS="$d" timeout 300 python scripts/wave_ab.py --config ${CFG:-C3} --kf ${KFS:-6,7} --reps ${REPS:-3} >> $OUT 2>&1
done
cat $OUT
