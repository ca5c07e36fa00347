#!/bin/bash
# A/B of an environment switch on one library, interleaved:  ENVS="TSAT_NO_SEG=1" SPECS="c4" bash scripts/ab_env.sh
cd "$(dirname "$0")/.."
O=gpurun_out/abenv; mkdir -p $O
for r in $(seq 1 ${ROUNDS:-2}); do
for spec in ${SPECS:-c4}; do
  cfg=${spec%@*}; n=""; [ "$spec" != "$cfg" ] && n="--n-per-gpu=${spec#*@}"
  for e in base ${ENVS}; do
    f=$O/${e//[^A-Za-z0-9_]/_}_${spec}_$r.json
    if [ "$e" = base ]; then envs=""; else envs="$e"; fi
    env $envs timeout 300 python bench.py --config $cfg $n --no-cpu --no-quality --no-e2e --no-extra --no-tts \
      --steps ${STEPS:-60} --warmup 20 > $f 2> $f.err
    echo -n "r$r $e $spec: "; python scripts/summarize_bench.py $f
  done
done
done
