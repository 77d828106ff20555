mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02r_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py tests/test_gpu_batch.py tests/test_gpu_persist.py -q -k "energy or compact or batch or persist" > gpurun_out/r02r_pytest_energy.log 2>&1
tail -3 gpurun_out/r02r_pytest_energy.log
timeout 300 python scripts/energy_time.py C1 C3 C4 > gpurun_out/r02r_energy.jsonl 2>&1; cat gpurun_out/r02r_energy.jsonl
timeout 600 python scripts/sweep.py --config C1 --kf 2,3,4,5,6,7 --rows 8,16,32,64 --reps 3 > gpurun_out/r02r_sweep_c1.jsonl 2>&1
timeout 600 python scripts/sweep.py --config C2 --kf 3,4,5,6,7 --rows 8,16,32,64 --reps 3 > gpurun_out/r02r_sweep_c2.jsonl 2>&1
python - <<'PY'
import json
for c in ("c1","c2"):
    rows=[json.loads(l) for l in open(f"gpurun_out/r02r_sweep_{c}.jsonl") if l.startswith("{")]
    rows.sort(key=lambda r:r["loop_ms"])
    for r in rows[:6]: print(c, r["kf"], r["rows"], round(r["loop_ms"],3), round(r["gpix_iter_s"],1), r["items"], r["launches"])
PY
