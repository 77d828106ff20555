mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ac_build.log 2>&1
for c in C0 C1 C2; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/r02ac_bench_$c.json 2> gpurun_out/r02ac_bench_$c.err; done
python - <<'PY'
import json
for c in ("C0","C1","C2"):
    try:
        b=json.loads(open(f"gpurun_out/r02ac_bench_{c}.json").read().strip().splitlines()[-1])
        cb=b.get("cpu_baseline") or {}
        print(c, round(b["value"],2), "cpu", cb.get("value"), cb.get("cores"), "1thr", cb.get("single_thread"))
    except Exception as e: print(c, "fail", e)
PY
