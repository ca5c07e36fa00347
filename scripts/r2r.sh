python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x --timeout=600 -k "row_block or peer or uni3_hub or uniform7 or lr_bound or fp64_state_variant or dense or long_clauses" > gpurun_out/r2r_pytest.txt 2>&1; tail -3 gpurun_out/r2r_pytest.txt
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for n in 128 256 512; do for env in "X=1" "TSAT_BLK_NOSORT=1"; do for mode in "" "--peer"; do
  env $env timeout 300 python bench.py --config c3 --n-per-gpu $n $mode $B > gpurun_out/s.json 2>/dev/null
  echo -n "N=$n $env $mode "; python scripts/summarize_bench.py gpurun_out/s.json
done; done; done
