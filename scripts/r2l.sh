python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -k "fp64" > gpurun_out/r2l_pytest.txt 2>&1; tail -30 gpurun_out/r2l_pytest.txt
