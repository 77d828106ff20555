# Warp-specialised stencil (k_stencil_ws): bitwise tests vs the single-warp kernel, then the
# C3 K-loop A/B (ws 0/1 alternating, k_fuse 6/7/8) and register-cap variants.
mkdir -p gpurun_out
OUT=gpurun_out/r02bb_ab.log
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bb_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ws.py -q -x > gpurun_out/r02bb_pytest_ws.log 2>&1
tail -3 gpurun_out/r02bb_pytest_ws.log >> $OUT
for dl in inf 0.2; do
  echo "delta=$dl" >> $OUT
  timeout 300 python scripts/sweep.py --kf 7 --rows 0 --delta $dl --reps 5 --ws 0,1,0,1 >> $OUT 2>&1
  timeout 300 python scripts/sweep.py --kf 6,8 --rows 0 --delta $dl --reps 5 --ws 1 >> $OUT 2>&1
done
for defs in "-DRDS_WS_MINB=4" "-DRDS_WS_MINB=6" "-DRDS_WS_NOWARM"; do
  d="${defs//,/ } -DRDS_KF_LIST(X)=X(6)X(7)X(8)"
  RDS_NVCC_DEFS="$d" python paper_1807_11534_b200/_build.py --force > /dev/null 2>>$OUT || { echo "build failed: $d" >> $OUT; continue; }
  grep -A2 "k_stencil_ws" paper_1807_11534_b200/build/ptxas.log | grep -E "Used|spill" >> $OUT
  RDS_NVCC_DEFS="$d" timeout 300 python scripts/sweep.py --kf 6,7,8 --rows 0 --delta inf --reps 5 --ws 1 >> $OUT 2>&1
done
cat $OUT
