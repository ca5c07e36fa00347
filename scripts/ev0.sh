set -x
O=gpurun_out/ev0
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python bench.py --config c4 --steps 60 --warmup 10 --no-cpu --no-quality --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c3 --steps 60 --warmup 10 --no-cpu --no-quality --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 2 -c 1 -o $O/prof_k_update_c4 -f python bench.py --config c4 --steps 10 --warmup 3 --no-e2e --no-cpu --no-quality > $O/ncu_c4.log 2>&1; tail -2 $O/ncu_c4.log
