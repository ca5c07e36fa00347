python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout=900 > gpurun_out/r2u_pytest.txt 2>&1; tail -2 gpurun_out/r2u_pytest.txt
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for rep in 1 2; do for cfg in c2 c3 c5:4096; do c=${cfg%%:*}; n=""; [ "$c" != "$cfg" ] && n="--n-per-gpu ${cfg##*:}"
for env in "X=1" "TSAT_NO_CW6=1"; do
  env $env timeout 300 python bench.py --config $c $n $B > gpurun_out/s.json 2>/dev/null; echo -n "$cfg $env "; python scripts/summarize_bench.py gpurun_out/s.json
done; done; done
VARIANTS="lib_c6_t832 lib_c6_t960" RUNS="c2" bash scripts/var2.sh
