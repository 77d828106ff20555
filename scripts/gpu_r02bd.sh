# 32-bit element-offset addressing (default) and the right-edge split of the march (EDGE):
# parity subset on the default build, then an alternating A/B of the C3 K-loop.
mkdir -p gpurun_out
OUT=gpurun_out/r02bd_ab.log
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bd_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ws.py tests/test_gpu_batch.py -q -x -k "ragged or fusion or skip_equiv or c0 or c1 or c2 or warm_start or schedules or frame or ws_ or batch" > gpurun_out/r02bd_pytest.log 2>&1
tail -2 gpurun_out/r02bd_pytest.log >> $OUT
for rep in 1 2; do
for defs in "-DRDS_ADDR64,-DRDS_EDGE_ALWAYS=1" "-DRDS_EDGE_ALWAYS=1" "-DRDS_ADDR64" "-DRDS_DEF=1"; do
  d="${defs//,/ } -DRDS_KF_LIST(X)=X(7)"
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>>$OUT || { echo "build failed: $d" >> $OUT; continue; }
  for dl in inf 0.2; do
    echo "rep=$rep defs=$defs delta=$dl" >> $OUT
    RDS_NVCC_DEFS="$d" timeout 300 python scripts/sweep.py --kf 7 --rows 0 --delta $dl --reps 5 --ws 0 >> $OUT 2>&1
  done
done; done
cat $OUT
