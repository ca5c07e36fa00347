# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on small step configurations
O=gpurun_out/${SAN_OUT:-san}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
CS="compute-sanitizer --print-limit 50 --target-processes all"
cat > /tmp/san_step.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2511_07737_b200 import Solver, config_default
from tsat_synth import planted_ksat, industrial_cnf, coloring_cnf
for name, cnf, N, ce in [("c1-like", planted_ksat(20, 85, 3, 1), 64, 0), ("blk128", planted_ksat(300, 1260, 3, 2), 128, 0),
                         ("ind7-1024", industrial_cnf(400, 1600, 3), 1024, 0), ("k15", coloring_cnf(10, 15, 3, 1), 256, 0),
                         ("dense", planted_ksat(256, 1075, 3, 2), 256, 1), ("c2-shape", planted_ksat(2000, 8400, 3, 1), 4096, 0),
                         ("fp64", industrial_cnf(300, 1100, 4), 512, 2), ("n8192-l2table", planted_ksat(100, 420, 3, 5), 8192, 0),
                         ("seg-k5-2048", planted_ksat(300, 900, 5, 2), 2048, 0), ("n8192-cluster", planted_ksat(100, 420, 3, 6), 8192, 3)]:
    import os
    if ce == 3: os.environ["TSAT_CLUSTER"] = "1"
    else: os.environ.pop("TSAT_CLUSTER", None)
    s = Solver(0)
    s.load_cnf(cnf)
    c = config_default(); c.clause_eval = 1 if ce == 1 else 0; c.state_fp64 = 1 if ce == 2 else 0
    s.init_batch(N, 3, c)
    info = s.step(3)
    s.export_best(4)
    s.close()
    print(name, "ok", info.best_unsat, flush=True)
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool python /tmp/san_step.py > $O/$tool.txt 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|ok " $O/$tool.txt | tail -8
done
TSAT_UPD_GRID=70 timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_peer.py -q -x -k "two_ranks and 1-256" -p no:cacheprovider > $O/memcheck_peer_w2.txt 2>&1; echo "peer rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $O/memcheck_peer_w2.txt | tail -4
