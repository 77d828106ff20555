mkdir -p gpurun_out
for m in 1 2 3; do
  export RDS_NVCC_DEFS="-DRDS_ENERGY_MINB=$m"
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ab_build.log 2>&1 || { echo build fail; continue; }
  echo "== MINB=$m"
  timeout 300 python scripts/energy_time.py C3 C4
done
