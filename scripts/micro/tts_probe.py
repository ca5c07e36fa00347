import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2511_07737_b200 import Solver, config_default
from tsat_synth import make_config, planted_ksat
for name, norm, steps in (("c2", 1, 720), ("c2", 0, 3600), ("c5@8192", 0, 3600)):
    if name == "c2":
        cnf, cfg = make_config("c2"); N = 4096
    else:
        cnf = planted_ksat(100_000, 425_000, 3, 1); N = 8192
    s = Solver(0); s.load_cnf(cnf)
    c = config_default(); c.normalize = norm
    s.init_batch(N, 1, c)
    t0 = time.time(); hist = []; gate = None
    for k in range(steps // 30):
        info = s.step(30)
        hist.append(info.best_unsat)
        if gate is None and info.best_unsat <= 0.01 * cnf.C: gate = info.t
        if info.solved: break
    print(name, "normalize", norm, "C", cnf.C, "gate(99%) step", gate, "solved", info.solved, info.solved_step,
          "final best", info.best_unsat, "trace", hist[::4], "%.1fs" % (time.time() - t0), flush=True)
