mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02h_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_persist.py tests/test_gpu_strips.py -x -q > gpurun_out/r02h_pytest_new.log 2>&1
tail -3 gpurun_out/r02h_pytest_new.log
timeout 600 python scripts/resident_ab.py > gpurun_out/r02h_paths.jsonl 2>&1
cat gpurun_out/r02h_paths.jsonl
for c in C1 C2; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-compact > gpurun_out/r02h_bench_$c.json 2>&1; done
python - <<'PY'
import json
for c in ("C1","C2"):
    try:
        b=json.loads(open(f"gpurun_out/r02h_bench_{c}.json").read().strip().splitlines()[-1])
        print(c, round(b["value"],1), [(p["delta_rel"], round(p["loop_ms"],3)) for p in b["per_delta"]])
    except Exception as e: print(c, "fail", e)
PY
