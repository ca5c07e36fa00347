# f4: dense path parity + timing + ncu of the dense and sparse clause kernels
O=gpurun_out/r2h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 -k "dense" > $O/pytest.txt 2>&1; tail -4 $O/pytest.txt
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for cfg in f4d f4s; do for ce in 0 1; do
  timeout 300 python bench.py --config $cfg --clause-eval $ce $B > $O/${cfg}_ce$ce.json 2>$O/err.txt; tail -2 $O/err.txt
  echo -n "$cfg ce=$ce "; python scripts/summarize_bench.py $O/${cfg}_ce$ce.json
done; done
for spec in "f4d 1 k_dense_clause" "f4d 0 k_clause" "f4s 1 k_dense_clause" "f4s 0 k_clause"; do
set -- $spec
timeout 600 ncu --set full --clock-control none -k regex:$3 -s 3 -c 1 -o $O/prof_$3_$1 -f python bench.py --config $1 --clause-eval $2 --no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 10 --warmup 3 > $O/ncu_$3_$1.log 2>&1; tail -1 $O/ncu_$3_$1.log
python scripts/ncu_summary.py $O $O/prof_$3_$1.ncu-rep > /dev/null 2>&1; head -20 $O/prof_$3_$1.txt
done
