mkdir -p gpurun_out
for d in "-DRDS_CHAINS=3" "-DRDS_MIDSPLIT -DRDS_CHAINS=3"; do
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>&1
  echo "== $d" >> gpurun_out/pytest_mid2.log
  timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3 >> gpurun_out/pytest_mid2.log
done
cat gpurun_out/pytest_mid2.log
TAG=mid2 VARIANTS="-DRDS_CHAINS=3 -DRDS_MIDSPLIT,-DRDS_CHAINS=3 -DRDS_MIDSPLIT" KFS=6,7 bash scripts/gpu_variants.sh
