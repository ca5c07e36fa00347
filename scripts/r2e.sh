# hybrid GPU -> CDCL time-to-SAT exploration
O=gpurun_out/r2e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
nproc
for spec in 400,1 500,1 500,2 600,1 1000,1 2000,1; do
  timeout 900 python bench.py --hybrid-only $spec > $O/hyb_$spec.json 2> $O/hyb_$spec.err; tail -2 $O/hyb_$spec.err; cat $O/hyb_$spec.json
done
