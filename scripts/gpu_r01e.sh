mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01e_pytest.log 2>&1; tail -2 gpurun_out/r01e_pytest.log
for c in C1 C2; do for d in inf 0.05; do timeout 300 python scripts/sweep.py --config $c --kf 3,4,5,6,7,8 --rows 0 --delta $d --reps 3; done; done > gpurun_out/r01e_kf_small.log 2>&1
cat gpurun_out/r01e_kf_small.log | cut -c1-160
