# Resident cluster (k_small) with the cluster barrier split into arrive / wait around the
# interior rows of phase A: its tests, then a same-box A/B against the tree at 9ebe161.
mkdir -p gpurun_out
OUT=$PWD/gpurun_out/r02bg_small_ab.log
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bg_build.log 2>&1
(cd _ab_old && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/r02bg_build_old.log 2>&1)
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -q -x -k "resident or c0 or frame" > gpurun_out/r02bg_pytest.log 2>&1
tail -1 gpurun_out/r02bg_pytest.log >> $OUT
for rep in 1 2 3; do for tree in . _ab_old; do
  echo "== $tree rep=$rep" >> $OUT
  (cd $tree && timeout 300 python scripts/small_time.py >> $OUT 2>&1)
done; done
cat $OUT
