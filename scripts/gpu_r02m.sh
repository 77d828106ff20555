mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02m_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "energy or compact or strips or batch" > gpurun_out/r02m_pytest.log 2>&1
tail -3 gpurun_out/r02m_pytest.log
timeout 300 python scripts/energy_time.py C3 C4 C1 > gpurun_out/r02m_energy.jsonl 2>&1
cat gpurun_out/r02m_energy.jsonl
