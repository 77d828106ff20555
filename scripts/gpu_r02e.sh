mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02e_build.log 2>&1
CMD="python scripts/wave_one.py --config C3 --kf 6"
$CMD > gpurun_out/r02e_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 1 -c 1 -o gpurun_out/r02e_wave $CMD > gpurun_out/r02e_ncu.log 2>&1
CMD2="python scripts/wave_one.py --config C3 --kf 6 --wave 0 --iters 60"
$CMD2 > gpurun_out/r02e_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 20 -c 1 -o gpurun_out/r02e_st66 $CMD2 > gpurun_out/r02e_ncu2.log 2>&1
ls -la gpurun_out | grep r02e
