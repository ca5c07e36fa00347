python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x --timeout=600 -k "industrial or hub or k7 or g_table or long_clauses or variants or c2_full or full_size" > gpurun_out/r2i_pytest.txt 2>&1; tail -3 gpurun_out/r2i_pytest.txt
VARIANTS="lib_noskip" RUNS="c2 c3 c4 c5:8192" bash scripts/var2.sh
