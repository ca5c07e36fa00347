# GPU test pass + smoke on one B200 (round 2)
O=gpurun_out/${TAG:-t}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout ${TMO:-1500} python -m pytest tests -m gpu -q -x --timeout=900 ${PYTEST_ARGS} > $O/pytest_gpu.txt 2>&1; tail -15 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -3 $O/smoke.txt
