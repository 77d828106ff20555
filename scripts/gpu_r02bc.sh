# Unrolled prologue with the warm-up stages above the cone elided (k_stencil_impl.cuh Act /
# Prologue): parity subset, then an alternating A/B of the C3 K-loop against RDS_NO_PROLOGUE.
mkdir -p gpurun_out
OUT=gpurun_out/r02bc_ab.log
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bc_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ws.py -q -x -k "ragged or fusion or skip_equiv or c0 or c1 or c2 or warm_start or schedules or frame or ws_" > gpurun_out/r02bc_pytest.log 2>&1
tail -2 gpurun_out/r02bc_pytest.log >> $OUT
for rep in 1 2; do
for defs in "-DRDS_NO_PROLOGUE" "-DRDS_P=1"; do
  d="${defs//,/ } -DRDS_KF_LIST(X)=X(5)X(6)X(7)X(8)"
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>>$OUT || { echo "build failed: $d" >> $OUT; continue; }
  for dl in inf 0.2; do
    echo "rep=$rep defs=$defs delta=$dl" >> $OUT
    RDS_NVCC_DEFS="$d" timeout 300 python scripts/sweep.py --kf 7 --rows 0 --delta $dl --reps 5 --ws 0 >> $OUT 2>&1
  done
  [ $rep = 1 ] && RDS_NVCC_DEFS="$d" timeout 300 python scripts/sweep.py --kf 5,6,8 --rows 0 --delta inf --reps 3 --ws 0 >> $OUT 2>&1
  [ $rep = 1 ] && RDS_NVCC_DEFS="$d" timeout 300 python scripts/sweep.py --config C1 --kf 7 --rows 0 --delta inf --reps 3 --ws 0 >> $OUT 2>&1
done; done
cat $OUT
