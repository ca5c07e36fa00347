python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for cfg in "c3 --n-per-gpu 256" "c3 --n-per-gpu 128" "c2"; do for env in "X=1" "TSAT_PEER_NOX=1"; do
  env $env timeout 300 python bench.py --config $cfg --peer $B > gpurun_out/s.json 2>/dev/null
  echo -n "$cfg $env peer "; python scripts/summarize_bench.py gpurun_out/s.json
done
timeout 300 python bench.py --config $cfg $B > gpurun_out/s.json 2>/dev/null; echo -n "$cfg fused "; python scripts/summarize_bench.py gpurun_out/s.json
done
