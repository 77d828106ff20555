# Final check with the prologue form on by default for images <= 2^22 px (TAG r02i): the whole
# GPU test suite, smoke, the default bench and bench.py on C0-C2.
T=r02i
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${T}_pytest.log 2>&1
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
: > gpurun_out/${T}_bench_configs.jsonl
for c in C0 C1 C2; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${T}_bench_configs.jsonl 2> gpurun_out/${T}_bench_$c.err
done
ls gpurun_out | grep $T
