# Evidence for the current tree on one B200: build, GPU tests, smoke, default bench line.
set -x
O=gpurun_out/${EV_OUT:-head}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
S=$(date +%s); timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$? secs=$(( $(date +%s)-S ))"
python - <<PY
import json; d=json.load(open("$O/bench_default.json")); r=d["roofline"]
print("c2 ms/step %.4f frac %.4f" % (d["ms_per_step"], r["frac"]))
for k, v in d.get("configs_more", {}).items(): print(k, v.get("ms_per_step"), {a: round(b, 4) for a, b in v.get("kernel_ms", {}).items()})
PY
