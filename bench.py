#!/usr/bin/env python
"""Benchmark: TurboSAT batched differentiable SAT step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One "step" = one full iteration of the hot path over
the whole candidate batch.  Metric (BASELINE.json): clause-candidate
evaluations per second = C * N_global * steps / s (plus gradient steps / s).
Workload at N=1: config c2 (planted random 3-SAT, V=10k, C=42k, ratio 4.2,
N=4096 candidates), seeded synthetic input.  The state streamed every step
(theta, m, v: 492 MB) is larger than L2, so no explicit flush is needed.

Prints ONE JSON line (rank 0).  Under torchrun (N>1) the candidate batch is
sharded over the ranks, the CNF is replicated, and per iteration the ranks
exchange Eq. 5's exact integer row / Jacobian sums and three maxima inside the
kernels over NVLink peer memory (or NCCL with --nccl).  Timed
on the device, max over ranks.  Scaling: c2 / c4 weak (N_config candidates
per GPU: BASELINE quotes them "on 1 B200"); c3 / c5 strong (BASELINE's fixed
global batch, 1024 / 65536 candidates split over the GPUs); --scaling
overrides.  At N=1 the line also carries the c3 / c4 sub-results
(configs_more), the time-to-SAT protocol on c2 (time_to_sat), trajectory
quality, the e2e pass and the oracle's CPU baseline.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=360)
    ap.add_argument("--warmup", type=int, default=30)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunk", type=int, default=30, help="iterations per tsat_step call (one CUDA graph)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-quality", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="W=1: run the candidate-sharded (multi-GPU) kernels")
    ap.add_argument("--nccl", action="store_true",
                    help="N>1: use the NCCL-exchange sharded path instead of the peer-exchange path (default)")
    ap.add_argument("--peer", action="store_true", help="W=1: run the peer-exchange kernels exchanging with themselves")
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="weak: N_config candidates per GPU; strong: N_config candidates in total (BASELINE's "
                         "fixed global batch; auto = strong for c3 / c5, weak otherwise)")
    ap.add_argument("--no-extra", action="store_true", help="skip the c3 / c4 sub-results (N=1)")
    ap.add_argument("--extra", default="c3,c4,c3@128,c5@8192",
                    help="configs timed as sub-results at N=1 (cfg@N: N candidates on this GPU)")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-SAT block (N=1)")
    ap.add_argument("--tts-config", default="c2")
    ap.add_argument("--tts-seeds", default="1,2,3,4,5")
    ap.add_argument("--tts-max-steps", type=int, default=3600)
    ap.add_argument("--tts-only", action="store_true", help="run only the time-to-SAT protocol and print it")
    ap.add_argument("--n-per-gpu", type=int, default=0, help="override the config's candidates per GPU (exploration)")
    ap.add_argument("--clause-eval", type=int, default=0, help="1: dense tensor-core clause evaluation (f4 experiment)")
    ap.add_argument("--trace", type=str, default="",
                    help="write a per-iteration CSV (iteration, lr, loss, best_unsat, best_fraction) of the first "
                         "--trace-steps iterations of this config to FILE (SPEC's --trace columns) and exit")
    ap.add_argument("--trace-steps", type=int, default=360)
    ap.add_argument("--hybrid-only", type=str, default="", help="V,seed[,N]: run only the GPU->CDCL hybrid time-to-SAT")
    return ap.parse_args()


def strong_scaling(args):
    return args.scaling == "strong" or (args.scaling == "auto" and args.config in ("c3", "c5"))


def upd_algorithmic_bytes(cnf, N):
    """SURVEY §8(d) bytes of k_update per launch: theta, m, v
    read + write, sign planes write + read, occurrence records, the g table."""
    V, K = cnf.V, cnf.K
    occ_words = int(np.sum(np.diff(cnf.clause_ptr) ** 2))
    return 24.0 * V * N + 2.0 * V * N / 8 + 4.0 * (occ_words + 2 * V + 1) + 8.0 * N * (K + 1)


def step_algorithmic_bytes(cnf, N):
    """SURVEY §8(d) per-step algorithmic bytes (whole step, one GPU)."""
    V, C, K = cnf.V, cnf.C, cnf.K
    b = 2 if K <= 3 else 3
    return 24.0 * V * N + 2.0 * V * N / 8 + 2.0 * C * N * b / 8 + 4.0 * (C + V + 2 * cnf.nnz + 2)


def time_config(name, local, stream, hbm, steps=30, warm=10):
    """Sub-result for another config on this GPU (N=1): device-timed steps and
    per-kernel CUDA-event times; k_update's fraction of the HBM roofline.
    "c3@128" = config c3 with 128 candidates on this GPU (one GPU's share of
    BASELINE's fixed global batch split over 8 GPUs)."""
    import torch
    from paper_2511_07737_b200 import Solver
    from tsat_synth import make_config
    base, _, nsh = name.partition("@")
    cnf, cfg = make_config(base)
    N = int(nsh) if nsh else cfg["N"]
    s = Solver(local, stream=stream)
    s.load_cnf(cnf)
    s.init_batch(N, cfg["seed"])
    chunk = 10
    for _ in range(warm // chunk):
        s.step(chunk, wait=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps // chunk):
        s.step(chunk, wait=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    s.set_profiling(True)
    s.kernel_times()
    for _ in range(steps // chunk):
        s.step(chunk, wait=False)
    torch.cuda.synchronize()
    kms, ks = s.kernel_times()
    s.close()
    names = ["k_clause", "k_gtable", "k_hub", "k_update", "k_step_end"]
    per = {n: float(kms[i] / ks) for i, n in enumerate(names)}
    ub = upd_algorithmic_bytes(cnf, N)
    sb = step_algorithmic_bytes(cnf, N)
    return {"workload": workload_desc(base, cnf, N) + (f" (one GPU's share of {cfg['N']} over {cfg['N'] // N} GPUs)"
                                                         if nsh else ""), "ms_per_step": ms, "value": cnf.C * N / (ms / 1e3),
            "unit": "evals/s", "steps": steps, "kernel_ms": per,
            "k_update": {"algorithmic_bytes": ub, "achieved_gbs": ub / (per["k_update"] / 1e3) / 1e9,
                         "frac": ub / (per["k_update"] / 1e3) / 1e9 / hbm},
            "step_algorithmic_bytes": sb, "step_frac": sb / (ms / 1e3) / 1e9 / hbm,
            "traffic_note": "ncu DRAM bytes of these kernels: profiles/ (static, per round)"}


def time_to_sat(name, seeds, max_steps, local, stream, chunk=30):
    """BASELINE.json's time-to-SAT: run each seed until some candidate reaches
    0 unsat (the library keeps its bits; verified on the host against the CNF)
    or max_steps; median steps / seconds over seeds, solved count, for the
    paper-exact reading (R3) and the f2 variants normalize-off and R28."""
    import torch
    from paper_2511_07737_b200 import Solver, config_default
    from tsat_synth import make_config
    _, cfg = make_config(name)
    N = cfg["N"]
    out = {"config": name, "N": N, "max_steps": max_steps, "seeds": seeds,
           "protocol": "run until a candidate has 0 unsat (model verified on the host) or max_steps; "
                       "instance seed = init seed = s"}
    for label, norm in (("paper_exact_R3", 1), ("normalize_off", 0), ("mean_magnitude_R28", 3)):
        runs = []
        for sd in seeds:
            cnf, _ = make_config(name, seed=sd)
            lits = np.asarray(cnf.lits)
            q = Solver(local, stream=stream)
            q.load_cnf(cnf)
            c = config_default()
            c.normalize = norm
            q.init_batch(N, sd, c)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            steps, solved, best = 0, False, None
            while steps < max_steps:
                inf = q.step(min(chunk, max_steps - steps))
                steps = inf.t
                best = inf.best_unsat if best is None else min(best, inf.best_unsat)
                if inf.solved:
                    solved = True
                    break
            wall = time.perf_counter() - t0
            rec = {"seed": sd, "solved": solved, "best_unsat": best, "steps_run": steps, "seconds": wall}
            if solved:
                sol = q.get_solution()
                vals, idx, st = sol
                var = np.abs(lits) - 1
                val = np.where(lits > 0, vals[var], 1 - vals[var])
                ok = bool((np.add.reduceat(val, cnf.clause_ptr[:-1]) > 0).all())
                rec.update(step_found=int(st), candidate=int(idx), verified=ok)
            q.close()
            runs.append(rec)
        sv = [r for r in runs if r["solved"]]
        out[label] = {"runs": runs, "solved": len(sv),
                      "median_steps_to_sat": float(np.median([r["step_found"] + 1 for r in sv])) if len(sv) * 2 > len(runs) else None,
                      "median_seconds_to_sat": float(np.median([r["seconds"] for r in sv])) if len(sv) * 2 > len(runs) else None,
                      "median_best_unsat": float(np.median([r["best_unsat"] for r in runs]))}
    return out


def hybrid_tts(cnf, N, seed, local, stream, threads, max_steps=3600, cdcl_limit_s=60.0, norms=(3, 1, 0)):
    """SURVEY f1 / PAPER.md §4.2 l.277-287: GPU gradient phase until the best
    candidate satisfies > 99 % of the clauses (or a model appears, or
    max_steps), then tsat_export_best (the best `threads` candidates, the
    paper's k = max(ceil(V/10^4), 20) most confident literals each) seeds a
    portfolio of CDCL instances on the host threads (plus one unseeded).
    Compared with the same CDCL run unseeded from scratch.  Wall-clock
    seconds, models verified on the host."""
    import torch
    from paper_2511_07737_b200 import Solver, cdcl_portfolio, cdcl_solve, config_default
    lits = np.asarray(cnf.lits)
    var = np.abs(lits) - 1

    def verify(m):
        val = np.where(lits > 0, m[var], 1 - m[var])
        return bool((np.add.reduceat(val, cnf.clause_ptr[:-1]) > 0).all())

    out = {"instance": f"V={cnf.V} C={cnf.C} (planted 3-SAT, seed {seed})", "N": N, "cdcl_threads": threads,
           "gate": "best candidate satisfies > 99% of clauses (PAPER.md l.279)"}
    t0 = time.perf_counter()
    r, m = cdcl_solve(cnf, conflict_limit=0, seed=0) if cdcl_limit_s <= 0 else \
        cdcl_portfolio(cnf, np.zeros((0, 0), np.int32), threads=1, unseeded=True, time_limit_s=cdcl_limit_s)
    out["cdcl_only"] = {"status": {10: "SAT", 20: "UNSAT", 0: "timeout"}[r.status], "seconds": time.perf_counter() - t0,
                        "conflicts": r.conflicts, "verified": verify(m) if m is not None else None,
                        "time_limit_s": cdcl_limit_s, "threads": 1}
    # the same thread count as the hybrid, no GPU seeds: a diversified portfolio
    # (randomised heuristics per instance, empty assumptions)
    t0 = time.perf_counter()
    r, m = cdcl_portfolio(cnf, np.zeros((threads, 1), np.int32), threads=threads, unseeded=True,
                          time_limit_s=cdcl_limit_s)
    out["cdcl_portfolio_unseeded"] = {"status": {10: "SAT", 20: "UNSAT", 0: "timeout"}[r.status],
                                      "seconds": time.perf_counter() - t0, "threads": threads,
                                      "verified": verify(m) if m is not None else None, "time_limit_s": cdcl_limit_s}
    labels = {1: "paper_exact_R3", 0: "normalize_off", 3: "mean_magnitude_R28"}
    for norm in norms:
        q = Solver(local, stream=stream)
        q.load_cnf(cnf)
        c = config_default()
        c.normalize = norm
        q.init_batch(N, seed, c)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        steps, gate, solved = 0, None, False
        while steps < max_steps:
            inf = q.step(10)
            steps = inf.t
            if inf.solved:
                solved = True
                break
            if (cnf.C - inf.best_unsat) / cnf.C > 0.99:
                gate = steps
                break
        t_gpu = time.perf_counter() - t0
        rec = {"gpu_steps": steps, "gpu_seconds": t_gpu, "gate_at_step": gate, "gpu_solved": solved}
        if solved:
            vals, idx, st = q.get_solution()
            rec.update(status="SAT (GPU)", verified=verify(vals), total_seconds=t_gpu)
        else:
            ex = q.export_best(threads)
            seeds = np.stack([e["lits"] for e in ex]).astype(np.int32)
            t_ex = time.perf_counter() - t0 - t_gpu
            r, m = cdcl_portfolio(cnf, seeds, threads=threads, unseeded=True, time_limit_s=cdcl_limit_s)
            rec.update(export_seconds=t_ex, k=int(seeds.shape[1]), best_unsat_exported=int(ex[0]["unsat"]),
                       status={10: "SAT", 20: "UNSAT", 0: "timeout"}[r.status], cdcl_seconds=r.seconds,
                       winner=("unseeded" if r.winner == -1 else int(r.winner)), failed_seeds=r.failed_seeds,
                       verified=verify(m) if m is not None else None,
                       total_seconds=time.perf_counter() - t0)
        q.close()
        out[labels[norm]] = rec
    return out


def quality_2v(cnf, N, seed, local, stream, iters=360):
    """Trajectory quality of the 2V-literal-row reading (tsat_synth.literal_split,
    PAPER.md l.191): the paper-exact Eq. 5 (R3) on 2V independent literal rows.
    Every 30 iterations the positive rows' bits (x_v = b of row v) are
    evaluated on the ORIGINAL CNF by a second solver (normalisation off, theta
    = +-1 from those bits, one evaluation step): best satisfied fraction of
    the original clauses, and the best of the relaxed (2V) problem."""
    from paper_2511_07737_b200 import Solver, config_default
    from tsat_synth import literal_split
    c2v = literal_split(cnf)
    q = Solver(local, stream=stream)
    q.load_cnf(c2v)
    q.init_batch(N, seed, config_default())
    ev = Solver(local, stream=stream)
    ev.load_cnf(cnf)
    ce = config_default()
    ce.normalize = 0
    ev.init_batch(N, seed, ce)
    best_orig, best_relaxed = None, None
    z = np.zeros((cnf.V, N), np.float32)
    for _ in range(iters // 30):
        inf = q.step(30)
        best_relaxed = inf.best_unsat if best_relaxed is None else min(best_relaxed, inf.best_unsat)
        words = q.debug(3, np.uint32, (c2v.V, N // 32))[:cnf.V]          # bit planes of the evaluated state
        bits = ((words[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(cnf.V, N)
        ev.set_state(np.where(bits > 0, 1.0, -1.0).astype(np.float32), z, z, 0)
        ev.step(1)
        u = int(ev.query_unsat().min())
        best_orig = u if best_orig is None else min(best_orig, u)
    q.close()
    ev.close()
    return {"iterations": iters, "best_unsat_original": best_orig,
            "best_satisfied_frac_original": (cnf.C - best_orig) / cnf.C,
            "best_unsat_relaxed_2V": best_relaxed,
            "note": "positive literal rows evaluated on the original CNF (the negative rows are not tied to them)"}


def workload_desc(name, cnf, N):
    kinds = {"c1": "planted random 3-SAT", "c2": "planted random 3-SAT", "c3": "planted random 3-SAT",
             "c4": "industrial-shaped CNF (lengths 2-7, power-law occurrences)", "c5": "planted random 3-SAT",
             "c2h": "2-hidden planted random 3-SAT (SURVEY f2 variant)",
             "f4d": "planted random 15-SAT, clause-dense (SURVEY f4 experiment)",
             "f4s": "planted random 3-SAT, small (SURVEY f4 experiment)"}
    return f"{name}: {kinds[name]} V={cnf.V} C={cnf.C} (ratio {cnf.C / cnf.V:.2f}), N={N} candidates"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                for line in out.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count()


def oracle_timing(cnf, N, seed, budget_s=20.0, min_steps=1, max_steps=None, omp=False):
    """Time the plain C oracle (as it stands; single thread, or its OpenMP
    build over all host cores) on a bounded sample: a slice of the candidate
    batch sized so the run takes ~budget_s."""
    from oracle import oracle as O
    O.use_openmp(omp)
    Ns = min(N, 256)
    o = O.Oracle(cnf, Ns, seed)
    t0 = time.perf_counter()
    o.step()
    one = time.perf_counter() - t0
    steps = max(min_steps, int(budget_s / max(one, 1e-6)))
    if max_steps:
        steps = min(steps, max_steps)
    # scale the sample to the budget: more candidates if one step is cheap
    if steps > 20 and Ns < N:
        Ns = min(N, int(Ns * min(steps / 20, N / Ns)) // 32 * 32 or 32)
        o = O.Oracle(cnf, Ns, seed)
        o.step()
        t0 = time.perf_counter()
        o.step()
        one = time.perf_counter() - t0
        steps = max(min_steps, int(budget_s / max(one, 1e-6)))
        if max_steps:
            steps = min(steps, max_steps)
    t0 = time.perf_counter()
    for _ in range(steps):
        o.step()
    el = time.perf_counter() - t0
    O.use_openmp(False)
    return dict(evals_per_s=cnf.C * Ns * steps / el, steps=steps, Ns=Ns, seconds=el,
                threads=O.omp_threads() if omp else 1)


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (this tier's reference arm) on the same
    config, rank 0 only, on host cores; each step a bounded candidate sample."""
    from tsat_synth import make_config
    if rank != 0:
        return
    cnf, cfg = make_config(args.config)
    N = cfg["N"] * max(1, world)
    model, cores = cpu_info()
    total_budget = 120.0
    per_step = total_budget / max(1, args.steps + args.warmup)
    from oracle import oracle as O
    O.use_openmp(True)                     # the oracle's OpenMP build over all host cores
    threads = O.omp_threads()
    Ns = 32
    o = O.Oracle(cnf, Ns, cfg["seed"])
    t0 = time.perf_counter()
    o.step()
    one = time.perf_counter() - t0
    Ns = int(max(32, min(N, Ns * per_step / max(one, 1e-6))) // 32 * 32)
    o = O.Oracle(cnf, Ns, cfg["seed"])
    for _ in range(args.warmup):
        o.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.step()
    el = time.perf_counter() - t0
    value = cnf.C * Ns * args.steps / el
    sample = f"{Ns} of {N} candidates per step (Eq. 5 mean over the sample), {args.steps} steps"
    line = {
        "impl": "reference", "metric": "clause-candidate evals/sec", "value": value, "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(args.config, cnf, N), "V": cnf.V, "C": cnf.C, "K": cnf.K,
                   "N_per_gpu": cfg["N"], "N_global": N, "seed": cfg["seed"],
                   "parallelism": f"CPU oracle (OpenMP build, {threads} threads) on a bounded candidate sample"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu": model, "host_cores": cores},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    from paper_2511_07737_b200 import Solver
    from tsat_synth import make_config

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    stream = torch.cuda.current_stream()
    if args.trace:
        if rank == 0:
            from paper_2511_07737_b200 import Solver, config_default
            from paper_2511_07737_b200.binding import lr_at
            from tsat_synth import make_config
            cnf, cfg = make_config(args.config)
            q = Solver(local, stream=stream)
            q.load_cnf(cnf)
            c = config_default()
            q.init_batch(args.n_per_gpu or cfg["N"], cfg["seed"], c)
            with open(args.trace, "w") as f:
                f.write("iteration,lr,loss,best_unsat,best_fraction\n")
                for it in range(args.trace_steps):
                    inf = q.step(1)                    # evaluates state `it`, then updates it
                    f.write(f"{it},{lr_at(c, it):.6g},{inf.loss:.10g},{inf.best_unsat},"
                            f"{(cnf.C - inf.best_unsat) / max(cnf.C, 1):.6f}\n")
            q.close()
            print(json.dumps({"trace": args.trace, "iterations": args.trace_steps}), flush=True)
        return
    if args.hybrid_only:
        if rank == 0:
            from tsat_synth import planted_ksat
            parts = [int(x) for x in args.hybrid_only.split(",")]
            V, sd = parts[0], parts[1]
            Nh = parts[2] if len(parts) > 2 else 4096
            cnf = planted_ksat(V, int(round(4.2 * V)), 3, sd)
            print(json.dumps({"metric": "hybrid time-to-SAT",
                              "hybrid": hybrid_tts(cnf, Nh, sd, local, stream, threads=max(1, (os.cpu_count() or 2) - 1))}),
                  flush=True)
        return
    if args.tts_only:
        if rank == 0:
            r = time_to_sat(args.tts_config, [int(x) for x in args.tts_seeds.split(",")], args.tts_max_steps, local,
                            stream)
            print(json.dumps({"metric": "time-to-SAT", "tts": r}), flush=True)
        return
    cnf, cfg = make_config(args.config)
    strong = strong_scaling(args)
    if strong and cfg["N"] % (32 * world):
        raise SystemExit(f"{args.config}: N = {cfg['N']} is not a multiple of 32 x {world}")
    N = cfg["N"] // world if strong else cfg["N"]       # candidates per GPU
    if args.n_per_gpu:
        N = args.n_per_gpu
    seed = cfg["seed"]

    use_peer = (world > 1 and not args.nccl) or args.peer
    peer_fallback = None

    def make_solver():
        if use_peer:           # exchanges inside the kernels over NVLink peer memory (CUDA IPC)
            return Solver(local, stream=stream, rank=rank, world=world, peer=True)
        if world > 1:
            return Solver.distributed(local, rank, world, stream=stream)
        if args.sharded:       # the multi-GPU kernels + NCCL on a 1-rank communicator
            from paper_2511_07737_b200 import nccl_unique_id
            return Solver(local, stream=stream, rank=0, world=1, nccl_unique_id=nccl_unique_id())
        return Solver(local, stream=stream)

    def load(sv):
        inf = sv.load_cnf(cnf)
        if use_peer:
            sv.connect_peers()
        return inf

    if world > 1 and use_peer:
        # the peer path needs CUDA IPC + peer access between the ranks' GPUs;
        # if any rank cannot set it up (or its first step fails), every rank
        # falls back to the NCCL-exchange path (same results, bit for bit)
        ok, why = 1, ""
        try:
            s = make_solver()
            info = load(s)
            s.init_batch(N * world, seed, **({'clause_eval': 1} if args.clause_eval else {}))
            s.step(1)
        except Exception as ex:  # noqa: BLE001
            ok, why = 0, f"{type(ex).__name__}: {ex}"[:200]
        flag = torch.tensor([ok], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            try:
                s.close()
            except Exception:  # noqa: BLE001
                pass
            use_peer = False
            peer_fallback = why or "another rank failed to set up the peer path"
            s = make_solver()
            info = load(s)
            s.init_batch(N * world, seed, **({'clause_eval': 1} if args.clause_eval else {}))
    else:
        s = make_solver()
        info = load(s)
        s.init_batch(N * world, seed, **({'clause_eval': 1} if args.clause_eval else {}))
    chunk = max(1, min(args.chunk, args.steps))
    assert args.steps % chunk == 0, "--steps must be a multiple of --chunk"
    # warm-up (also instantiates the chunk-sized CUDA graph)
    w = max(3, args.warmup)
    wk = 0
    while wk < w:
        s.step(chunk, wait=False)
        wk += chunk
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- timed region (device events on the library's stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps // chunk):
            s.step(chunk, wait=False)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    last = s.get_info()
    evals = float(cnf.C) * N * world * args.steps
    value = evals / (ms / 1000.0)

    # ---- second timed pass with per-kernel CUDA events (roofline)
    s.set_profiling(True)
    s.kernel_times()
    for _ in range(args.steps // chunk):
        s.step(chunk, wait=False)
    torch.cuda.synchronize()
    kms, ksteps = s.kernel_times()
    s.set_profiling(False)
    names = ["k_clause", "k_gtable", "k_hub", "k_update", "k_step_end"]
    per = {n: float(kms[i] / ksteps) for i, n in enumerate(names)}
    upd_bytes = upd_algorithmic_bytes(cnf, N)
    upd_ms = per["k_update"]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = upd_bytes / (upd_ms / 1000.0) / 1e9
    traffic, traffic_src = None, None
    try:      # dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture (profiles/)
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[args.config]["k_update"]
        traffic = tr["bytes"]
        traffic_src = ("profiles/" + tr["report"] + " (static: one ncu --set full capture of this build, "
                       "refreshed per round with scripts/ncu_summary.py; not measured in this run)")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": "k_update", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                "algorithmic_bytes_per_launch": upd_bytes, "kernel_ms": per,
                "kernel_share": {n: per[n] / sum(per.values()) for n in names}}

    kps = s.kernels_per_step()
    s.close()                                 # the e2e solver below needs the memory (c5: 100 GB each)
    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # the one-time setup (load + init + graph capture) inside the timed
        # region is amortised over at least one LR cycle (360 steps), however
        # few steps the device-timed line uses
        K_e2e = max(args.steps, 360)
        s2 = make_solver()
        # the caller's pinned host buffers (allocated once, like the workspace's owner would)
        pins = [torch.empty(N, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        pnp = [p.numpy() for p in pins]      # host views of the pinned buffers (no torch op per step)
        evs = [torch.cuda.Event() for _ in range(2)]
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        f0 = torch.cuda.Event(enable_timing=True); f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        load(s2)                              # host CSR -> device
        tl = time.perf_counter()
        s2.init_batch(N * world, seed, **({'clause_eval': 1} if args.clause_eval else {}))
        ti = time.perf_counter()
        s2.step(1)                            # first call: captures + instantiates the 1-step graph
        ts = time.perf_counter()
        s2.query_unsat_async(pins[1].data_ptr())
        torch.cuda.synchronize()
        best_seen = int(pnp[1].min())
        setup_ms = (time.perf_counter() - t0) * 1000.0
        setup_parts = {"load_ms": (tl - t0) * 1e3, "init_ms": (ti - tl) * 1e3, "first_step_ms": (ts - ti) * 1e3,
                       "query_sync_ms": setup_ms - (ts - t0) * 1e3}
        # every step: H2D of its step scalars (pinned), D2H of its per-candidate
        # unsat counts into a pinned double buffer; step t's counts are read on
        # the host while step t + 1 runs (tsat_query_unsat_async)
        for i in range(K_e2e - 1):
            s2.step(1, wait=False)
            s2.query_unsat_async(pins[i & 1].data_ptr())
            evs[i & 1].record(stream)
            if i > 0:
                evs[(i - 1) & 1].synchronize()
                b = int(pnp[(i - 1) & 1].min())
                best_seen = b if best_seen is None else min(best_seen, b)
        evs[(K_e2e - 2) & 1].synchronize()
        b = int(pnp[(K_e2e - 2) & 1].min())
        best_seen = b if best_seen is None else min(best_seen, b)
        f1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms_e2e = max(f0.elapsed_time(f1), wall * 1000.0)
        if world > 1:
            t = torch.tensor([ms_e2e], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
        cnf_bytes = 8 * (cnf.C + 1) + 4 * cnf.nnz
        e2e = {"value": float(cnf.C) * N * world * K_e2e / (ms_e2e / 1000.0), "unit": "evals/s",
               "h2d_bytes_per_step": cnf_bytes / K_e2e + 64, "d2h_bytes_per_step": 4 * N,
               "steps": K_e2e, "best_unsat_seen": best_seen, "setup_ms_in_timed_region": setup_ms,
               "setup_parts": setup_parts,
               "includes": "load_clauses + init_batch + per step: tsat_step(1) (H2D step scalars) + "
                           "tsat_query_unsat_async into pinned memory, read on the host during the next step"}
        s2.close()

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = oracle_timing(cnf, N, seed, budget_s=12.0, omp=True)
        r1 = oracle_timing(cnf, N, seed, budget_s=8.0)
        model, cores = cpu_info()
        cpu = {"value": r["evals_per_s"], "unit": "evals/s", "cores": r["threads"], "kind": "oracle",
               "sample": f"{r['steps']} oracle steps on {r['Ns']} of {N} candidates ({r['seconds']:.1f} s, "
                         f"OpenMP build over {r['threads']} threads)",
               "single_thread": {"value": r1["evals_per_s"], "cores": 1,
                                 "sample": f"{r1['steps']} steps on {r1['Ns']} candidates ({r1['seconds']:.1f} s)"},
               "cpu": model, "host_cores": cores}

    # ---- sub-results: the other single-GPU BASELINE configs (device-timed)
    extra = None
    if world == 1 and not args.no_extra:
        extra = {}
        for name in [x for x in args.extra.split(",") if x and x != args.config]:
            try:
                extra[name] = time_config(name, local, stream, hbm)
            except Exception as ex:  # noqa: BLE001
                extra[name] = {"error": f"{type(ex).__name__}: {ex}"[:200]}
    tts = None
    if world == 1 and not args.no_tts:
        tts = time_to_sat(args.tts_config, [int(x) for x in args.tts_seeds.split(",")], args.tts_max_steps, local,
                          stream)

    # ---- GPU -> CPU CDCL hand-off (f1): hybrid time-to-SAT on a planted
    # instance small enough for the CDCL arms to be timed (V = 600)
    hybrid = None
    if world == 1 and not args.no_tts:
        from tsat_synth import planted_ksat
        hybrid = hybrid_tts(planted_ksat(600, 2520, 3, 1), 4096, 1, local, stream,
                            threads=max(1, (os.cpu_count() or 2) - 1), cdcl_limit_s=20.0)

    # ---- trajectory quality (not a timing): one LR cycle (360 iterations) of
    # the paper-exact Eq. 5 reading (R3) and of the normalize-off variant;
    # best satisfied fraction and whether the 99 % gate fires
    quality = None
    if world == 1 and not args.no_quality:
        from paper_2511_07737_b200 import config_default
        quality = {"iterations": 360, "gate": "best candidate satisfies > 99% of clauses"}
        for label, norm in (("paper_exact_R3", 1), ("normalize_off", 0), ("mean_magnitude_R28", 3)):
            q = Solver(local, stream=stream)
            q.load_cnf(cnf)
            c = config_default()
            c.normalize = norm
            q.init_batch(N, seed, c)
            best, gate = None, None
            for _ in range(12):
                inf = q.step(30)
                best = inf.best_unsat if best is None else min(best, inf.best_unsat)
                if gate is None and (cnf.C - inf.best_unsat) / cnf.C > 0.99:
                    gate = inf.t
            quality[label] = {"best_unsat": best, "best_satisfied_frac": (cnf.C - best) / cnf.C,
                              "gate_99_at_iteration": gate, "solved": bool(inf.solved)}
            q.close()
        quality["literal_rows_2V_R3"] = quality_2v(cnf, N, seed, local, stream)

    line = {
        "metric": "clause-candidate evals/sec", "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": w, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(args.config, cnf, N * world), "V": cnf.V, "C": cnf.C, "K": cnf.K,
                   "N_per_gpu": N, "N_global": N * world, "seed": seed,
                   "parallelism": (f"candidate-sharded x{world}, exact exchanges inside the kernels over NVLink peer "
                                   "memory" if world > 1 and use_peer else
                                   f"candidate-sharded x{world} (NCCL exact int64 exchanges)" if world > 1 else
                                   "single GPU, peer-exchange kernels (self)" if args.peer else
                                   "single GPU, sharded kernels on a 1-rank NCCL communicator" if args.sharded else
                                   "single GPU"),
                   "l2": "state (theta, m, v: %.0f MB) larger than L2; no flush" % (12 * cnf.V * N / 1e6),
                   "graph_chunk": chunk, "peer_fallback": peer_fallback},
        "gradient_steps_per_s": args.steps / (ms / 1000.0),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": kps * args.steps, "clocks": clk.summary(),
        "last_info": {"t": last.t, "best_unsat": last.best_unsat, "loss": last.loss, "solved": last.solved},
        "quality": quality, "configs_more": extra, "time_to_sat": tts, "hybrid_time_to_sat": hybrid,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
