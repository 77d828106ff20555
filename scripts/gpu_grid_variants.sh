mkdir -p gpurun_out
for defs in "-DRDS_GRID_PROFILE" "-DRDS_GRID_PROFILE -DRDS_GRID_ALLPOLL"; do
  export RDS_NVCC_DEFS="$defs"
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/gv_build.log 2>&1 || { echo build fail "$defs"; tail gpurun_out/gv_build.log; continue; }
  timeout 120 python scripts/grid_one.py C1 2>&1 | tail -12
  timeout 120 python scripts/grid_one.py 256x1024 2>&1 | tail -12
done
