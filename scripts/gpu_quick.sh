# quick round trip: build, the GPU parity tests selected by $TESTK, benches of $CONFIGS (k_update share + ms/step)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -k "${TESTK:-ragged or industrial or hub or chunked or sharded or variants or c1 or export or full_size}" 2>&1 | tail -15
for C in ${CONFIGS:-c2 c4}; do
timeout 900 python bench.py --config $C --steps 60 --warmup 30 --no-cpu --no-quality --no-e2e > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; tail -3 gpurun_out/bench_$C.err
python - <<PY
import json; d=json.load(open("gpurun_out/bench_$C.json")); r=d["roofline"]
print("$C", "ms/step %.4f" % d["ms_per_step"], "frac %.4f" % r["frac"], {k: round(v, 4) for k, v in r["kernel_ms"].items()})
PY
done
