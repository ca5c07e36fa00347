# Round evidence on one B200: parity tests, smoke, the default bench line (c2), c3/c4/c5 bench lines,
# the ncu launch list of the bench command, one ncu --set full capture per hot kernel and config.
set -x
O=gpurun_out/ev
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 2>&1 | tail -30 > $O/pytest_gpu.txt; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 > $O/smoke.txt; cat $O/smoke.txt
timeout 900 python bench.py --steps 120 --warmup 30 > $O/bench_c2.json 2> $O/bench_c2.err; tail -2 $O/bench_c2.err
for C in c3 c4 c5 c2h; do
Q=--no-quality; [ $C = c2h ] && Q=; timeout 900 python bench.py --config $C --steps 60 --warmup 10 --no-cpu $Q > $O/bench_$C.json 2> $O/bench_$C.err; tail -2 $O/bench_$C.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c2.csv python bench.py --steps 30 --warmup 30 --no-e2e --no-cpu --no-quality > /dev/null 2>&1
for spec in "c2 k_update" "c2 k_clause" "c2 k_gtable" "c3 k_update" "c4 k_update" "c4 k_clause" "c4 k_hub"; do
set -- $spec
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o $O/prof_$2_$1 -f python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-quality > $O/ncu_$2_$1.log 2>&1; tail -1 $O/ncu_$2_$1.log
done
