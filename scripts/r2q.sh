python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x --timeout=600 -k "row_block or peer or uni3_hub or uniform7 or lr_bound or fp64_state_variant" > gpurun_out/r2q_pytest.txt 2>&1; tail -3 gpurun_out/r2q_pytest.txt
RUNS="c3:128 c3:256 c3:512" bash scripts/var2.sh
EXTRA="--peer" RUNS="c3:128 c3:256" bash scripts/var2.sh
