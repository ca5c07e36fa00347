O=gpurun_out/r2g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 -k "g_table or chunked or c2_full" > $O/pytest.txt 2>&1; tail -5 $O/pytest.txt
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for n in 8192 4096; do
for env in "TSAT_NO_GS_GLOBAL=1" "X=1"; do
  env $env TSAT_GEOM_VERBOSE=1 timeout 300 python bench.py --config c5 --n-per-gpu $n $B > $O/c5_$n_$env.json 2>$O/err.txt; grep -h geometry $O/err.txt | head -1
  python scripts/summarize_bench.py $O/c5_$n_$env.json
done; done
