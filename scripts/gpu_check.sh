# GPU round check: parity tests, smoke, bench, ncu launch list + one full capture of k_update.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 ${PYTEST_ARGS} 2>&1 | tail -60 > gpurun_out/pytest_gpu.txt; tail -60 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --steps 120 --warmup 30 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 30 --warmup 30 --no-e2e --no-cpu --no-quality > /dev/null 2>&1; tail -6 gpurun_out/launches.csv
if [ -n "$NCU_FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 -o gpurun_out/prof_update -f python bench.py --steps 30 --warmup 30 --no-e2e --no-cpu --no-quality > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_clause -s 3 -c 1 -o gpurun_out/prof_clause -f python bench.py --steps 30 --warmup 30 --no-e2e --no-cpu --no-quality > gpurun_out/ncu_full2.log 2>&1; tail -3 gpurun_out/ncu_full2.log
fi
