# One full ncu capture per hot kernel (1 GPU), reports left in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
CFG=${CFG:-c2}
for K in ${KERNELS:-k_update k_clause}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c 1 -o gpurun_out/prof_${K}_${CFG} -f python bench.py --config $CFG --steps 30 --warmup 30 --no-e2e --no-cpu --no-quality > gpurun_out/ncu_${K}.log 2>&1; tail -3 gpurun_out/ncu_${K}.log
done
