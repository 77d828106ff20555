# 3-D step with two barriers per plane step (RDS_VOL_2BAR) vs three: the 3-D tests on the 2BAR
# build, then an alternating A/B of bench3d.py (V1 256^3, K = 200).
mkdir -p gpurun_out
OUT=gpurun_out/r02bk_vol_ab.log
: > $OUT
RDS_NVCC_DEFS="-DRDS_VOL_2BAR" python paper_1807_11534_b200/_build.py > /dev/null 2>&1
RDS_NVCC_DEFS="-DRDS_VOL_2BAR" timeout 900 python -m pytest tests/test_gpu_vol.py -q -x > gpurun_out/r02bk_pytest_vol.log 2>&1
tail -1 gpurun_out/r02bk_pytest_vol.log >> $OUT
for rep in 1 2 3; do for d in "-DRDS_VOL_3BAR=1" "-DRDS_VOL_2BAR"; do
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py > /dev/null 2>&1
  RDS_NVCC_DEFS="$d" timeout 600 python scripts/bench3d.py 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('$d rep=$rep', d['delta_rel'], round(d['ms'], 3), round(d['gvoxel_iter_s'], 1), round(d['hbm_roofline']['frac'], 3))
" >> $OUT
done; done
cat $OUT
