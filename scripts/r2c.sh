# round 2: row-block kernel parity + small-N benches
O=gpurun_out/r2c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x --timeout=600 -k "row_block or peer or uniform7 or uni3_hub or lr_bound" > $O/pytest.txt 2>&1; tail -15 $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for n in 128 256 512; do
  for mode in "" "--peer"; do
    TSAT_GEOM_VERBOSE=1 timeout 600 python bench.py --config c3 --n-per-gpu $n $mode $B > $O/c3_n${n}${mode}.json 2>$O/err.txt; grep -h geometry $O/err.txt | head -1; grep -v geometry $O/err.txt | tail -3
    python - <<PY
import json; d=json.load(open("$O/c3_n${n}${mode}.json")); r=d["roofline"]
print("c3 N=$n $mode", "ms/step %.3f" % d["ms_per_step"], "frac %.3f" % r["frac"], {k: round(v, 3) for k, v in r["kernel_ms"].items()})
PY
  done
done
