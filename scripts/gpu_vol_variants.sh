# Compile-time variants of the 3-D step kernel (RDS_NVCC_DEFS; VOL_DEFS overrides the list):
# parity of each build (tests/test_gpu_vol.py) and V1 timing (scripts/bench3d.py).
mkdir -p gpurun_out
: > gpurun_out/vol_variants.log
for d in ${VOL_DEFS:-"-DRDS_VOL_TY=16 -DRDS_VOL_TY=32 -DRDS_VOL_TY=8"}; do
  d="${d//,/ }"
  RDS_NVCC_DEFS="$d -DRDS_KF_LIST(X)=X(4)X(7)" python paper_1807_11534_b200/_build.py --force > /dev/null 2>&1
  echo "== $d" >> gpurun_out/vol_variants.log
  timeout 600 python -m pytest tests/test_gpu_vol.py -q -x 2>&1 | tail -1 >> gpurun_out/vol_variants.log
  timeout 300 python scripts/bench3d.py >> gpurun_out/vol_variants.log 2>&1
done
cat gpurun_out/vol_variants.log | cut -c1-220
