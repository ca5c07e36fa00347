python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x --timeout=600 -k "g_table or chunked or c2_full or ragged or peer_w1 or sharded or hub" > gpurun_out/r2o_pytest.txt 2>&1; tail -3 gpurun_out/r2o_pytest.txt
TSAT_GEOM_VERBOSE=1 RUNS="c5:8192 c2 c4" bash scripts/var2.sh
grep -h geometry gpurun_out/var/base_c5*.err | head -2
