mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ad_build.log 2>&1
for d in 0.05 0.1 0.2 0.4; do
  timeout 600 python scripts/sweep.py --config C2 --kf 3,4,5,6,7 --rows 0,8,16,32 --delta $d --reps 3 > gpurun_out/r02ad_sweep_c2_$d.jsonl 2>&1
  timeout 600 python scripts/sweep.py --config C1 --kf 3,4,5,7 --rows 0,8,16 --delta $d --reps 3 > gpurun_out/r02ad_sweep_c1_$d.jsonl 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02ad_sweep_*.jsonl")):
    rows=[json.loads(l) for l in open(f) if l.startswith("{")]
    if not rows: print(f, "empty"); continue
    rows.sort(key=lambda r:r["loop_ms"])
    d=[r for r in rows if r["kf"]==7 and r["rows"]==0]
    print(f.split("/")[-1], "best", [(r["kf"], r["rows"], round(r["loop_ms"],3)) for r in rows[:3]], "default(7,0)", round(d[0]["loop_ms"],3) if d else None)
PY
