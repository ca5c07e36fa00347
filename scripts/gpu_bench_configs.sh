# bench on the larger configs (no CPU baseline: the oracle would take minutes per step there)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for C in ${CONFIGS:-c3 c4}; do
timeout 900 python bench.py --config $C --steps 60 --warmup 30 --no-cpu > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; tail -3 gpurun_out/bench_$C.err; cat gpurun_out/bench_$C.json | cut -c1-1500
done
