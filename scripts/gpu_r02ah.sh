mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ah_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q -k "resident or c0 or ragged" > gpurun_out/r02ah_pytest.log 2>&1
tail -5 gpurun_out/r02ah_pytest.log
for ll in 0 1; do
  echo "== RDS_SMALL_LL=$ll"
  RDS_SMALL_LL=$ll timeout 300 python scripts/resident_ab.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['case'], d['delta_rel'], 'resident', round(d.get('resident_solve_ms', -1), 4), 'stencil', round(d.get('stencil_solve_ms', -1), 4))
"
done
