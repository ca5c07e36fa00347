"""Where the e2e setup time goes (c2): load, workspace, init, first step (graph capture), later steps."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, numpy as np
from paper_2511_07737_b200 import Solver
from tsat_synth import make_config
cnf, cfg = make_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
N = cfg["N"]
torch.cuda.synchronize()
for rep in range(3):
    s = Solver(0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.load_cnf(cnf); torch.cuda.synchronize(); t1 = time.perf_counter()
    nb = s.workspace_bytes(N); t1b = time.perf_counter()
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda"); torch.cuda.synchronize(); t1c = time.perf_counter()
    del ws
    s.init_batch(N, 1); torch.cuda.synchronize(); t2 = time.perf_counter()
    s.step(1); torch.cuda.synchronize(); t3 = time.perf_counter()
    s.step(1); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms  ws_bytes {1e3*(t1b-t1):.2f}  torch.empty {1e3*(t1c-t1b):.2f}  init {1e3*(t2-t1c):.2f} ms  "
          f"first step {1e3*(t3-t2):.2f} ms  second step {1e3*(t4-t3):.2f} ms", flush=True)
    s.close()
