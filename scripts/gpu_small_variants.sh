# Timing experiments of the resident-cluster kernel (k_small.cu) via RDS_NVCC_DEFS.
mkdir -p gpurun_out
OUT=gpurun_out/small_variants_${TAG:-x}.log
: > $OUT
for defs in ${VARIANTS:-"-DRDS_SMALL_X"}; do
  d="${defs//,/ }"
  echo "== $d" >> $OUT
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>>$OUT || { echo "build failed: $d" >> $OUT; continue; }
  RDS_NVCC_DEFS="$d" timeout 300 python scripts/resident_ab.py >> $OUT 2>&1
done
cat $OUT
