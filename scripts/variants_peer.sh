# variants.sh for the peer-exchange kernels at W = 1 (bench --peer)
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-c2}; do
  for v in base ${VARIANTS}; do
    if [ "$v" = base ]; then lib=paper_2511_07737_b200/libturbosat.so; else lib=paper_2511_07737_b200/$v.so; fi
    TSAT_LIB=$PWD/$lib timeout 300 python bench.py --peer --config $cfg --no-cpu --no-quality --no-e2e --steps 120 \
      > gpurun_out/varp_${v}_${cfg}.json 2> gpurun_out/varp_${v}_${cfg}.err
    echo -n "$v "; python scripts/summarize_bench.py gpurun_out/varp_${v}_${cfg}.json
  done
done
