set -x
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 > $O/pytest_gpu.txt 2>&1; tail -15 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -3 $O/smoke.txt
S=$(date +%s); timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$? secs=$(( $(date +%s)-S ))"; tail -5 $O/bench_default.err; cat $O/bench_default.json
