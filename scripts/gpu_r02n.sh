mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02n_pytest.log 2>&1
tail -5 gpurun_out/r02n_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n_smoke.log 2>&1
tail -3 gpurun_out/r02n_smoke.log
timeout 900 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
python - <<'PY'
import json
b=json.loads(open("gpurun_out/r02n_bench.json").read().strip().splitlines()[-1])
print(b["value"], b["ms_per_step"], b["roofline"]["frac"], b["clocks"], b["e2e"]["value"], b["cpu_baseline"]["value"])
print([(p["delta_rel"], p["path"], round(p["loop_ms"],2)) for p in b["per_delta"]])
PY
