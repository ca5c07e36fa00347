# peer kernels at W = 1 (self exchange) vs the fused kernel, and a library variant: bash scripts/peer_ab.sh lib_x
for r in $(seq 1 ${ROUNDS:-2}); do
for v in base $1; do
  if [ "$v" = base ]; then lib=paper_2511_07737_b200/libturbosat.so; else lib=paper_2511_07737_b200/$v.so; fi
  for p in "" "--peer"; do
    TSAT_LIB=$PWD/$lib timeout 300 python bench.py --config ${CFG:-c2} $p --no-cpu --no-quality --no-e2e --no-extra --no-tts --steps 60 --warmup 20 > gpurun_out/peer_${v}_$r.json 2>/dev/null
    echo -n "r$r $v ${p:-fused}: "; python scripts/summarize_bench.py gpurun_out/peer_${v}_$r.json
  done
done
done
