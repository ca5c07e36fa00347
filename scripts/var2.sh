# A/B of compile-time variants on one box: VARIANTS="lib_a lib_b" RUNS="c3 c3:128" bash scripts/var2.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/var
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for run in ${RUNS:-c2}; do
  cfg=${run%%:*}; n=""; [ "$cfg" != "$run" ] && n="--n-per-gpu ${run##*:}"
  for v in base ${VARIANTS}; do
    if [ "$v" = base ]; then lib=paper_2511_07737_b200/libturbosat.so; else lib=paper_2511_07737_b200/$v.so; fi
    f=gpurun_out/var/${v}_${cfg}${run##*:}.json
    TSAT_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg $n $B $EXTRA > $f 2> $f.err
    python - "$f" "$v $run" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1])); r = d["roofline"]
    print(sys.argv[2], "ms/step %.4f" % d["ms_per_step"], "k_update %.4f frac %.4f" % (r["kernel_ms"]["k_update"], r["frac"]), "k_clause %.4f" % r["kernel_ms"]["k_clause"])
except Exception as e:
    print(sys.argv[2], "FAILED", e, open(sys.argv[1] + ".err").read()[-500:])
PY
  done
done
