#!/bin/bash
# Time compile-time variants of libturbosat side by side on one box:
#   VARIANTS="lib_v1 lib_v2" CFGS="c2" bash scripts/variants.sh
# Each paper_2511_07737_b200/<name>.so must have been built here first
# (build.build(out=..., defines=(...))).  Default library = "base".
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CFGS:-c2}; do
  for v in base ${VARIANTS}; do
    if [ "$v" = base ]; then lib=paper_2511_07737_b200/libturbosat.so; else lib=paper_2511_07737_b200/$v.so; fi
    TSAT_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --no-cpu --no-quality --no-e2e \
      > gpurun_out/var_${v}_${cfg}.json 2> gpurun_out/var_${v}_${cfg}.err
    echo -n "$v "; python scripts/summarize_bench.py gpurun_out/var_${v}_${cfg}.json
  done
done
