# f4 dense tensor-core path parity + f4 configs + KB=8 thread variants + c5 shards
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 -k "dense or tau_final or variants" > $O/pytest.txt 2>&1; tail -12 $O/pytest.txt
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for cfg in f4d f4s; do for ce in 0 1; do
  timeout 300 python bench.py --config $cfg --clause-eval $ce $B > $O/${cfg}_ce$ce.json 2>$O/err.txt; tail -2 $O/err.txt
  python scripts/summarize_bench.py $O/${cfg}_ce$ce.json 2>/dev/null || python -c "import json;d=json.load(open('$O/${cfg}_ce$ce.json'));print('$cfg ce=$ce', d['ms_per_step'], d['roofline']['kernel_ms'])"
done; done
VARIANTS="lib_t8_640 lib_t8_768" RUNS="c4" bash scripts/var2.sh
RUNS="c5:8192 c5" bash scripts/var2.sh
