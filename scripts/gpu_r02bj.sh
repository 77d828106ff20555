# Prologue form as a separate instantiation (RDS_OPT_PROLOGUE): bitwise tests, then an
# alternating A/B (off / on) of the K-loop on C1, C2, C3 and C4.
mkdir -p gpurun_out
OUT=gpurun_out/r02bj_ab.log
: > $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bj_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_prologue.py -q -x > gpurun_out/r02bj_pytest.log 2>&1
tail -1 gpurun_out/r02bj_pytest.log >> $OUT
for c in C1 C2 C3; do for dl in inf 0.2; do
  timeout 600 python scripts/sweep.py --config $c --kf 7 --rows 0 --delta $dl --reps 5 --pro 0,1,0,1 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('$c', '$dl', 'pro', d['pro'], round(d['loop_ms'], 4), d['items'])
" >> $OUT
done; done
timeout 900 python scripts/sweep.py --config C4 --kf 7 --rows 0 --delta 0.2 --reps 2 --pro 0,1 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('C4 0.2 pro', d['pro'], round(d['loop_ms'], 3), d['items'])
" >> $OUT
cat $OUT
