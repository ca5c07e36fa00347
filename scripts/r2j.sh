python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x --timeout=600 -k "row_block or peer or g_table or uni3_hub or uniform7 or long_clauses or dense" > gpurun_out/r2j_pytest.txt 2>&1; tail -3 gpurun_out/r2j_pytest.txt
VARIANTS="lib_old lib_noskip" RUNS="c2 c3 c3:128 c4" bash scripts/var2.sh
