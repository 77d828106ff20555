set -x
python -m pytest tests -m gpu -x -q -k "parity or tol or fusion" > gpurun_out/pdl_pytest.log 2>&1; tail -2 gpurun_out/pdl_pytest.log
for cfg in C1 C2 C3 C4; do
  for pdl in 1 0; do
    if [ $pdl = 0 ]; then export RDS_NO_PDL=1; else unset RDS_NO_PDL; fi
    python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/pdl_${cfg}_$pdl.json 2>gpurun_out/pdl_${cfg}_$pdl.err
    python -c "import json;d=json.load(open('gpurun_out/pdl_${cfg}_$pdl.json'));print('$cfg pdl=$pdl',d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])"
  done
done
unset RDS_NO_PDL
python scripts/tol_overhead.py > gpurun_out/pdl_tol.log 2>&1; tail -12 gpurun_out/pdl_tol.log
