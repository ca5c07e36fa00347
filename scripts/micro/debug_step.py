import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import oracle as O
from tsat_synth import planted_ksat
from paper_2511_07737_b200 import Solver
cnf = planted_ksat(400, 1680, 3, 12); N = 256
s = Solver(0); s.load_cnf(cnf); s.init_batch(N, 21)
o = O.Oracle(cnf, N, 21)
s.set_state(o.theta, o.m, o.v, 0)
th0 = o.theta.copy(); m0 = o.m.copy(); v0 = o.v.copy()
s.step(1); ref = o.step()
th, m, v, t = s.get_state()
for name, a, b in (("theta", th, o.theta), ("m", m, o.m), ("v", v, o.v)):
    bad = np.argwhere(a != b)
    print(name, "mismatch", len(bad))
    for (i, j) in bad[:5]:
        print("  v=%d n=%d gpu=%r ora=%r grad=%r th0=%r m0=%r v0=%r" % (i, j, a[i, j], b[i, j], ref.grad[i, j], th0[i, j], m0[i, j], v0[i, j]))
print("unsat equal", np.array_equal(s.query_unsat(), ref.unsat))
