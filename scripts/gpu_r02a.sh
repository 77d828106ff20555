# Round 2, call a: MUFU error bounds (exhaustive), fixed MUFU throughput rows, the GPU tests
# with the stated-K parity additions (timed), smoke, the default bench.
mkdir -p gpurun_out
nproc > gpurun_out/r02a_nproc.txt; lscpu | grep -i "model name" >> gpurun_out/r02a_nproc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_err scripts/micro/mufu_err.cu && timeout 120 /tmp/mufu_err > gpurun_out/r02a_mufu_err.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_tput scripts/micro/mufu_tput.cu && timeout 120 /tmp/mufu_tput > gpurun_out/r02a_mufu_tput.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02a_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s --durations=25 > gpurun_out/r02a_pytest.log 2>&1
tail -3 gpurun_out/r02a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02a_ref.json 2> gpurun_out/r02a_ref.err
cat gpurun_out/r02a_mufu_err.txt
