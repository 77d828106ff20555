mkdir -p gpurun_out
RDS_NVCC_DEFS="-DRDS_MIDSPLIT" python paper_1807_11534_b200/_build.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -5 > gpurun_out/pytest_mid.log; tail -3 gpurun_out/pytest_mid.log
TAG=mid VARIANTS="-DRDS_MIDSPLIT -DRDS_MIDSPLIT,-DRDS_CHAINS=3 -DRDS_MIDSPLIT,-DRDS_CHAINS=3,-DRDS_DEN_SCALAR -DRDS_CHAINS=3,-DRDS_DEN_SCALAR" KFS=6,7 bash scripts/gpu_variants.sh
