import os, sys, time; sys.path.insert(0, os.getcwd())
import torch
from paper_2511_07737_b200 import Solver
from tsat_synth import make_config
cnf, cfg = make_config("c2"); N = cfg["N"]
def run(tag, steps, chunk, st=None, prof=False):
    kw = {} if st is None else {"stream": st}
    s = Solver(0, **kw); s.load_cnf(cnf); s.init_batch(N, 1)
    for _ in range(steps // chunk): s.step(chunk)
    torch.cuda.synchronize()
    if prof:
        s.set_profiling(True)
        for _ in range(steps // chunk): s.step(chunk, wait=False)
        torch.cuda.synchronize()
        s.kernel_times()
        s.set_profiling(False)
    s.close()
    pins = torch.empty(N, dtype=torch.int32, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s2 = Solver(0, **kw); ta = time.perf_counter()
    s2.load_cnf(cnf); torch.cuda.synchronize(); tl = time.perf_counter()
    s2.init_batch(N, 1); torch.cuda.synchronize(); ti = time.perf_counter()
    s2.step(1); th = time.perf_counter(); torch.cuda.synchronize(); ts = time.perf_counter()
    s2.query_unsat_async(pins.data_ptr()); torch.cuda.synchronize(); tq = time.perf_counter()
    s2.step(1); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{tag}: create {1e3*(ta-t0):.2f} load {1e3*(tl-ta):.2f} init {1e3*(ti-tl):.2f} step1 {1e3*(ts-ti):.2f} (host {1e3*(th-ti):.2f}) query {1e3*(tq-ts):.2f} step2 {1e3*(t2-tq):.2f}", flush=True)
    s2.close()
run("after 390 steps chunk 30", 390, 30)
run("again", 390, 30)
run("after 30 steps chunk 1", 30, 1)
run("torch current stream", 390, 30, torch.cuda.current_stream())
run("after a profiling pass", 390, 30, torch.cuda.current_stream(), prof=True)
run("after a profiling pass again", 390, 30, torch.cuda.current_stream(), prof=True)
