# A/B of a kernel (default k_update) between the base library and variants: instructions, time, issue
# activity, stall latencies, L2 hit rate, DRAM bytes (one launch each, ncu cold-cache replay)
CFG=${CFG:-c2}
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then lib=paper_2511_07737_b200/libturbosat.so; else lib=paper_2511_07737_b200/$v.so; fi
  TSAT_LIB=$PWD/$lib timeout 600 ncu --clock-control none -k regex:${KERNEL:-k_update} -s 3 -c 1 --csv \
    --log-file gpurun_out/ab_$v.csv \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_no_instruction.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum \
    python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu --no-quality ${BENCH_ARGS} > /dev/null 2>&1
  python - "$v" gpurun_out/ab_$v.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 5]
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    print(sys.argv[1], d.get("Metric Name"), d.get("Metric Unit"), d.get("Metric Value"))
PY
done
