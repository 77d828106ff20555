mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02an_build.log 2>&1
python scripts/vol_one.py > gpurun_out/r02an_vol_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vol_step2 -s 25 -c 1 -o gpurun_out/r02an_vol_step2 python scripts/vol_one.py > gpurun_out/r02an_ncu_vol.log 2>&1
ls gpurun_out | grep r02an
