set -x
nproc; nvidia-smi -L; lscpu | grep -E 'Model name|^CPU\(s\)'
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -40 > gpurun_out/pytest1.log; tail -40 gpurun_out/pytest1.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -5
for kf in 1 3 5 7 8; do timeout 300 python bench.py --kf $kf --steps 2 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -2; done > gpurun_out/kfsweep.log
cat gpurun_out/kfsweep.log
