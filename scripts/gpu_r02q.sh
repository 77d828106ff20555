mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02q_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_vol.py -q > gpurun_out/r02q_pytest_vol.log 2>&1
tail -3 gpurun_out/r02q_pytest_vol.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py tests/test_gpu_batch.py -q -k "energy or compact or batch" > gpurun_out/r02q_pytest_energy.log 2>&1
tail -3 gpurun_out/r02q_pytest_energy.log
timeout 300 python scripts/energy_time.py C3 C4 > gpurun_out/r02q_energy.jsonl 2>&1; cat gpurun_out/r02q_energy.jsonl
RDS_VOL_RPT=1 timeout 300 python scripts/bench3d.py > gpurun_out/r02q_bench3d_rpt1.jsonl 2>&1
timeout 300 python scripts/bench3d.py > gpurun_out/r02q_bench3d_rpt2.jsonl 2>&1
cat gpurun_out/r02q_bench3d_rpt1.jsonl gpurun_out/r02q_bench3d_rpt2.jsonl
for c in C0 C1 C2 C4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02q_bench_$c.json 2>&1; done
python - <<'PY'
import json
for c in ("C0","C1","C2","C4"):
    try:
        b=json.loads(open(f"gpurun_out/r02q_bench_{c}.json").read().strip().splitlines()[-1])
        print(c, round(b["value"],1), round(b["roofline"]["frac"],3) if b["roofline"] else None, [(p["delta_rel"], p["path"], round(p["loop_ms"],3)) for p in b["per_delta"]])
        print("   compact:", [(p["delta_rel"], p["path"], round(p["speedup_vs_full"],2)) for p in (b.get("restricted_compact") or {}).get("per_delta", [])])
    except Exception as e: print(c, "fail", e)
PY
