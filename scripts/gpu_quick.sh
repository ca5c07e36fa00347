python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -k "ragged or industrial or hub or chunked or sharded or variants or c1 or export or full_size" 2>&1 | tail -15
CONFIGS="c4" bash scripts/gpu_bench_configs.sh 2>&1 | tail -5
