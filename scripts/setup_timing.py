import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, numpy as np
from paper_2511_07737_b200 import Solver
from tsat_synth import make_config
cnf, cfg = make_config("c2")
torch.cuda.synchronize()
for rep in range(3):
    s = Solver(0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.load_cnf(cnf); torch.cuda.synchronize(); t1 = time.perf_counter()
    s.init_batch(4096, 1); torch.cuda.synchronize(); t2 = time.perf_counter()
    s.step(1); torch.cuda.synchronize(); t3 = time.perf_counter()
    s.step(1); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms  init {1e3*(t2-t1):.2f} ms  first step {1e3*(t3-t2):.2f} ms  second step {1e3*(t4-t3):.2f} ms")
    s.close()
