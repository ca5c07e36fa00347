#!/bin/bash
# A/B of library builds on one box, interleaved (base, variants, base, ...) per config:
#   VARIANTS="lib_head" SPECS="c2 c4 c3@128" ROUNDS=2 TESTK="..." bash scripts/ab.sh
# Each paper_2511_07737_b200/<name>.so must exist (build.build(out=...)); base = libturbosat.so.
cd "$(dirname "$0")/.."
O=gpurun_out/ab; mkdir -p $O
if [ -n "$TESTK" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -k "$TESTK" 2>&1 | tail -4
fi
for r in $(seq 1 ${ROUNDS:-2}); do
for spec in ${SPECS:-c2}; do
  cfg=${spec%@*}; n=""; [ "$spec" != "$cfg" ] && n="--n-per-gpu=${spec#*@}"
  for v in base ${VARIANTS}; do
    if [ "$v" = base ]; then lib=paper_2511_07737_b200/libturbosat.so; else lib=paper_2511_07737_b200/$v.so; fi
    f=$O/${v}_${spec}_$r.json
    TSAT_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg $n --no-cpu --no-quality --no-e2e --no-extra --no-tts \
      --steps ${STEPS:-60} --warmup 20 > $f 2> $O/${v}_${spec}_$r.err
    echo -n "r$r $v $spec: "; python scripts/summarize_bench.py $f
  done
done
done
