# round 2: small-N candidate shards (strong-scaling shares) and k_update ncu captures at c3/c4
O=gpurun_out/r2b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for n in 128 256 512; do
  for mode in "" "--peer"; do
    timeout 600 python bench.py --config c3 --n-per-gpu $n $mode $B > $O/c3_n${n}${mode}.json 2>$O/err.txt; tail -2 $O/err.txt
    python - <<PY
import json; d=json.load(open("$O/c3_n${n}${mode}.json")); r=d["roofline"]
print("c3 N=$n $mode", "ms/step %.3f" % d["ms_per_step"], "frac %.3f" % r["frac"], {k: round(v, 3) for k, v in r["kernel_ms"].items()})
PY
  done
done
for spec in "c4 k_update" "c3 k_update"; do
set -- $spec
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o $O/prof_$2_$1 -f python bench.py --config $1 $B > $O/ncu_$2_$1.log 2>&1; tail -1 $O/ncu_$2_$1.log
python scripts/ncu_lines.py $O/prof_$2_$1.ncu-rep 60 > $O/lines_$2_$1.txt 2>&1
ncu -i $O/prof_$2_$1.ncu-rep --page source --csv --print-source sass > $O/sass_$2_$1.csv 2>/dev/null
done
ls -la $O
