mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q 2>&1 | tail -8 > gpurun_out/pytest_slow.log; tail -3 gpurun_out/pytest_slow.log
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py --smoke > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.log
