python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x --timeout=600 -k "row_block or peer or c1 or ragged or lr_bound or variants or enumeration or fig1 or dense" > gpurun_out/r2m_pytest.txt 2>&1; tail -3 gpurun_out/r2m_pytest.txt
VARIANTS="lib_keep220 lib_keep220_f50" RUNS="c5:8192 c2 c3:128" bash scripts/var2.sh
