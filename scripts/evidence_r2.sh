# Round-2 evidence on one B200: GPU tests, smoke, default bench line, reference arm, f4 timing,
# ncu launch list of the bench command, ncu --set full per hot kernel/config (summaries + traffic json).
set -x
O=gpurun_out/${EV_OUT:-ev2}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
S=$(date +%s); timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$? secs=$(( $(date +%s)-S ))"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; cat $O/bench_reference.json | head -c 400
B="--no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 30 --warmup 10"
for cfg in f4d f4s; do for ce in 0 1; do
  timeout 300 python bench.py --config $cfg --clause-eval $ce $B > $O/${cfg}_ce$ce.json 2>/dev/null
  echo -n "$cfg ce=$ce "; python scripts/summarize_bench.py $O/${cfg}_ce$ce.json
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 30 --warmup 30 $B > /dev/null 2>&1
cp profiles/ncu_traffic.json /tmp/ncu_traffic_before.json
for spec in "c2 k_update c2" "c3 k_update c3" "c4 k_update c4" "c3 k_update_blk c3n128 --n-per-gpu=128" "c5 k_update c5n8192 --n-per-gpu=8192" "c2 k_clause c2" "c4 k_clause_seg c4" "c4 k_hub c4" ${EXTRA_NCU}; do
set -- $spec
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2[<(]" -s 2 -c 1 -o $O/prof_$2_$3 -f python bench.py --config $1 $4 --no-e2e --no-cpu --no-quality --no-extra --no-tts --steps 10 --warmup 3 > $O/ncu_$2_$3.log 2>&1; tail -1 $O/ncu_$2_$3.log
python scripts/ncu_summary.py $O $O/prof_$2_$3.ncu-rep > /dev/null 2>&1
python scripts/ncu_lines.py $O/prof_$2_$3.ncu-rep 40 > $O/lines_$2_$3.txt 2>&1
done
cp profiles/ncu_traffic.json $O/ncu_traffic.json
rm -f $O/*.ncu-rep
[ -n "$SANITIZE" ] && SAN_OUT=${EV_OUT:-ev2}/san bash scripts/sanitize.sh     # (compute-sanitizer is closed on the pool)
CFG=c2 bash scripts/peer_ab.sh > $O/peer_c2.txt 2>&1; cat $O/peer_c2.txt
ls $O
