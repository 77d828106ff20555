mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ag_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_compact.py -x -q > gpurun_out/r02ag_pytest_compact.log 2>&1
tail -15 gpurun_out/r02ag_pytest_compact.log
timeout 600 python scripts/compact_sweep.py --config C3 --deltas 0.02 0.05 0.1 0.2 > gpurun_out/r02ag_compact_c3.jsonl 2>&1
timeout 300 python scripts/compact_sweep.py --config C2 --deltas 0.02 0.05 0.1 0.2 > gpurun_out/r02ag_compact_c2.jsonl 2>&1
timeout 300 python scripts/compact_sweep.py --config C1 --deltas 0.02 0.05 0.1 0.2 > gpurun_out/r02ag_compact_c1.jsonl 2>&1
python - <<'PY'
import json
for c in ("c3","c2","c1"):
    for ln in open(f"gpurun_out/r02ag_compact_{c}.jsonl"):
        try: d=json.loads(ln)
        except Exception: print(ln.strip()); continue
        print(c, d["delta_rel"], round(d["rd_frac"],3), "dense", round(d["dense_loop_ms"],2), "compact", round(d["compact_loop_ms"],2), "x_full", round(d["speedup_compact_vs_full"],2), d["same_u"])
PY
