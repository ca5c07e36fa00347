python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q -x --timeout=900 > gpurun_out/r2v_pytest.txt 2>&1; tail -2 gpurun_out/r2v_pytest.txt
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 60 --warmup 10"
for env in "X=1" "TSAT_NO_CW6=1" "X=1" "TSAT_NO_CW6=1"; do
  env $env timeout 300 python bench.py --config c2 $B > gpurun_out/s.json 2>/dev/null; echo -n "c2 $env "; python scripts/summarize_bench.py gpurun_out/s.json
done
