python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for rep in 1 2; do
for g in 6 5 4; do
  TSAT_UPD_MAXGROUPS=$g timeout 300 python bench.py --config c5 --n-per-gpu 8192 $B > gpurun_out/g$g.json 2>/dev/null
  echo -n "groups=$g "; python scripts/summarize_bench.py gpurun_out/g$g.json
done; done
