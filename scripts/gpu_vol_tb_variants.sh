mkdir -p gpurun_out
for defs in "-DRDS_VTB_TY=32" "-DRDS_VTB_MINB=2" "-DRDS_VTB_TY=16" "-DRDS_VTB_TY=16 -DRDS_VTB_MINB=3"; do
  export RDS_NVCC_DEFS="$defs"
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/vtb_build.log 2>&1 || { echo build fail "$defs"; continue; }
  echo "== $defs"
  timeout 300 python scripts/bench3d.py --kf 2,3 --reps 3 | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['kf'], d['delta_rel'], round(d['gvoxel_iter_s'],1), d['kz'])
"
done
