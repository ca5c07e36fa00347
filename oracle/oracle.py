"""TEST INFRASTRUCTURE ONLY - Python driver for the plain C oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It sequences the C
functions of ``tsat_oracle.c`` into one TurboSAT iteration in the paper's
order (Fig. 3, §3.2, §4.1):

  Eq. 5 normalise -> Eq. 2 binarise -> Eq. 1 R = PA -> §3.1.4 hard S / unsat
  -> Eq. 4 SmoothMin, Eq. 3 loss -> STE backward (P^T) -> Eq. 5 Jacobian
  -> AdamW with the §4.1 LR schedule.

Selection and export (§4.2) are a stable sort here
(numpy.lexsort), the plain definition.

Sharding: every cross-candidate reduction (Q, I, gmax, thmax, S, best) goes
through ``self.comm`` (``LocalComm``: identity).  tests/ substitute a
torch.distributed (gloo) or thread-barrier communicator to prove that a
candidate-sharded run equals the unsharded one.
"""
from __future__ import annotations

import ctypes as ct
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tsat_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -ffp-contract=off): the single-thread
    library and the OpenMP build of the same source (liboracle_omp.so)."""
    for out, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
            tmp = out + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, out)
    return _LIB


_lib = None
_lib_omp = None
_use_omp = False


def use_openmp(enabled: bool = True, threads: int | None = None) -> None:
    """Route every oracle call through the OpenMP build (all host cores, or
    `threads`).  Results are identical to the single-thread build."""
    global _use_omp
    _use_omp = bool(enabled)
    if threads:
        os.environ["OMP_NUM_THREADS"] = str(int(threads))


def omp_threads() -> int:
    """Threads the OpenMP build uses (OMP_NUM_THREADS, else all cores)."""
    return int(os.environ.get("OMP_NUM_THREADS", "0") or 0) or (os.cpu_count() or 1)


def lib():
    global _lib, _lib_omp
    if _use_omp:
        if _lib_omp is None:
            build()
            _lib_omp = _bind(ct.CDLL(_LIB_OMP))
        return _lib_omp
    if _lib is None:
        _lib = _bind(ct.CDLL(build()))
    return _lib


def _bind(L):
    """Declare the C signatures on a loaded oracle library."""
    P = ct.c_void_p
    i32, i64, u64, f64, f32 = ct.c_int, ct.c_int64, ct.c_uint64, ct.c_double, ct.c_float
    sig = {
        "or_philox4x32_10": (None, [P, P, P]),
        "or_init": (None, [i32, i64, i32, u64, P, P, P]),
        "or_row_sums": (i32, [i32, i32, P, P]),
        "or_row_sums_abs": (i32, [i32, i32, P, P]),
        "or_row_finish": (None, [i32, i64, P, i32, f64, P, P, P, P]),
        "or_binarize": (None, [i32, i32, P, P, P]),
        "or_clause_eval": (None, [i32, P, P, i32, P, P]),
        "or_histogram": (None, [i32, i32, i32, P, P]),
        "or_smoothmin": (None, [i32, i32, P, P, f64, P, P, P]),
        "or_smoothmin_direct": (f64, [i32, P, f64]),
        "or_backward": (None, [i32, i32, P, P, i32, i32, P, P, P]),
        "or_jacobian_partial": (None, [i32, i32, P, P, P, i64, f64, f32, P, P, P]),
        "or_jacobian_finish": (None, [i32, i64, P, P, P, P, P, i32, P, P]),
        "or_grad": (None, [i32, i32, P, P, P, P]),
        "or_grad_mag": (None, [i32, i32, P, P, P, P, P]),
        "or_lr_at": (f64, [i64, f64, f64, i32, i32, f64]),
        "or_adamw": (None, [i32, i64, i32, P, P, P, P, i64, i64, f64, f64, f64, f64, f64, f64, u64]),
        "or_abs_max": (f32, [ct.c_size_t, P]),
        "or_gmax": (f64, [i32, i32, P, P]),
        "or_hist_stream": (None, [i32, P, P, i32, i32, P, P, P]),
        "or_backward_rows": (None, [i32, P, P, i32, i32, P, P, P, i32, P, P, P]),
        "or_init64": (None, [i32, i64, i32, u64, P, P, P]),
        "or_row_sums64": (i32, [i32, i32, P, P, P, i32]),
        "or_row_finish64": (None, [i32, i64, P, P, i32, f64, P, P, P, P]),
        "or_binarize64": (None, [i32, i32, P, P, P]),
        "or_backward64": (None, [i32, i32, P, P, i32, i32, P, P, P]),
        "or_jacobian_partial64": (None, [i32, i32, P, P, P, i64, f64, f64, P, P, P]),
        "or_grad64": (None, [i32, i32, P, P, P, P, i32, P]),
        "or_adamw64": (None, [i32, i64, i32, P, P, P, P, i64, i64, f64, f64, f64, f64, f64, f64, u64]),
        "or_abs_max64": (f64, [ct.c_size_t, P]),
        "or_gmax64": (f64, [i32, i32, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ct.c_void_p)


# ---------------------------------------------------------------- pieces
def philox(ctr, key):
    c = np.array(ctr, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def init_theta(V, N, seed, n0=0, Nl=None):
    Nl = N if Nl is None else Nl
    th = np.empty((V, Nl), np.float32)
    m = np.empty((V, Nl), np.float32)
    v = np.empty((V, Nl), np.float32)
    lib().or_init(V, n0, Nl, seed, _p(th), _p(m), _p(v))
    return th, m, v


def lr_at(t, cfg):
    return lib().or_lr_at(t, cfg.lr0, cfg.decay_factor, cfg.decay_every, cfg.restart_every, cfg.lr_min)


def adam_step(t, cfg):
    """(moments reset at t?, bias-correction step).  Variant:
    with reset_moments_on_restart the AdamW optimiser is re-created at every
    LR restart (t > 0, t mod restart_every = 0), as a fresh torch.optim.AdamW
    would be: m = v = 0 and its step count starts again at 1."""
    if not cfg.reset_moments_on_restart:
        return False, t + 1
    return (t > 0 and t % cfg.restart_every == 0), t % cfg.restart_every + 1


def clause_eval(cnf, b):
    Nl = b.shape[1]
    R = np.empty((cnf.C, Nl), np.uint8)
    lib().or_clause_eval(cnf.C, _p(cnf.clause_ptr), _p(cnf.lits), Nl, _p(np.ascontiguousarray(b, np.uint8)), _p(R))
    return R


def histogram(R, K):
    C, Nl = R.shape
    h = np.empty((Nl, K + 1), np.int32)
    lib().or_histogram(C, Nl, K, _p(R), _p(h))
    return h


def exp_table(tau, K):
    """E[d] = exp(-tau d), d = 0..K (host libm; R11)."""
    return np.array([math.exp(-tau * d) for d in range(K + 1)], dtype=np.float64)


def smoothmin(h, tau):
    Nl, K1 = h.shape
    K = K1 - 1
    E = exp_table(tau, K)
    S = np.empty(Nl, np.float64)
    g = np.empty((Nl, K1), np.float64)
    rmin = np.empty(Nl, np.int32)
    lib().or_smoothmin(Nl, K, _p(np.ascontiguousarray(h, np.int32)), _p(E), tau, _p(S), _p(g), _p(rmin))
    return S, g, rmin


def tau_at(t: int, cfg) -> float:
    """SmoothMin temperature of iteration t (Eq. 4's tau).  The paper fixes
    none (R1: constant tau).  Variant R29 (tau_final > 0): geometric from tau
    at the start of each LR cycle to tau_final at its
    last iteration: tau (tau_final / tau)^((t mod R) / (R - 1))."""
    if cfg.tau_final > 0 and cfg.restart_every > 1:
        return cfg.tau * math.pow(cfg.tau_final / cfg.tau, (t % cfg.restart_every) / (cfg.restart_every - 1))
    return cfg.tau


def smoothmin_direct(col, tau):
    c = np.ascontiguousarray(col, np.int32)
    return lib().or_smoothmin_direct(len(c), _p(c), tau)


def backward(cnf, R, g32):
    """g32: the fp32 derivative table (R26)."""
    Nl = R.shape[1]
    K = g32.shape[1] - 1
    G = np.empty((cnf.V, Nl), np.float64)
    g32 = np.ascontiguousarray(g32, np.float32)
    lib().or_backward(cnf.V, cnf.C, _p(cnf.clause_ptr), _p(cnf.lits), Nl, K, _p(R), _p(g32), _p(G))
    return G


def compute_k(V: int) -> int:
    """k = 0.01% of V, at least 20, at most V (R13 ceil)."""
    return min(V, max(-(-V // 10000), 20))


def select_top(unsat: np.ndarray, M: int, n0: int = 0):
    """Top-M candidates by (unsat asc, index asc) (R15)."""
    idx = np.arange(len(unsat), dtype=np.int64) + n0
    order = np.lexsort((idx, unsat))
    return idx[order[:M]], unsat[order[:M]]


def export_partial(absG_col: np.ndarray, bits_col: np.ndarray, k: int):
    """k variables with smallest |G| (ties -> lower v), most confident first
    (R14, R15).  Returns signed 1-based DIMACS literals."""
    v = np.arange(len(absG_col), dtype=np.int64)
    order = np.lexsort((v, absG_col))[:k]
    lits = np.where(bits_col[order] == 1, order + 1, -(order + 1)).astype(np.int32)
    return lits, absG_col[order]


# ---------------------------------------------------------------- config
@dataclass
class Config:
    tau: float = 1.0
    normalize: int = 1          # 0 off (R20), 1 Eq. 5 global (R3), 2 per shard, 3 mean magnitude (R28)
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 1e-2
    lr0: float = 1e-1
    lr_min: float = 1e-15
    decay_factor: float = 10.0
    decay_every: int = 30
    restart_every: int = 360
    noise_sigma: float = 0.0
    eps_norm: float = 1e-8
    reset_moments_on_restart: int = 0
    tau_final: float = 0.0      # > 0: SmoothMin temperature annealed within each LR cycle (variant f2, R29)
    state_fp64: int = 0         # 1: theta, m, v and every fp32 rounding of R6/R13/R26/R27 in fp64 (variant f2, R30)


class LocalComm:
    """Single-shard communicator: every reduction is the identity."""

    def sum_i64(self, a):
        return a

    def max(self, x):
        return x

    def min_key(self, k):
        return k

    def gather_f64(self, a):
        return a


@dataclass
class StepOut:
    t: int
    bits: np.ndarray          # evaluated state b_t (V x Nl, uint8)
    R: np.ndarray             # C x Nl
    h: np.ndarray             # Nl x (K+1)
    unsat: np.ndarray         # Nl
    S: np.ndarray             # Nl
    g: np.ndarray             # Nl x (K+1) fp64 (Eq. 4 derivative)
    g32: np.ndarray           # Nl x (K+1) fp32 table used by the backward (R26)
    loss: float               # -sum_n S_n over ALL candidates
    G: np.ndarray             # V x Nl pre-Jacobian variable gradient, fp32 values (R27) held in fp64
    grad: np.ndarray          # V x Nl fp32 (post-Jacobian)
    J: np.ndarray
    d: np.ndarray
    gmax: float
    thmax: float
    best_unsat: int
    best_idx: int
    lr: float
    extra: dict = field(default_factory=dict)


def binary_problem_matrix(cnf):
    """The rows of P (§3.1.1, l.143-149): P is a 0/1 matrix, so a literal
    repeated inside a clause is ONE entry (its column holds a 1).  Returns a
    clause list with repeated literals removed (first occurrence kept); a
    clause holding x and ~x keeps both (two distinct columns)."""
    from tsat_synth import Cnf
    out = []
    changed = False
    for cl in cnf.clauses():
        seen, row = set(), []
        for x in cl:
            if x not in seen:
                seen.add(x)
                row.append(x)
        changed |= len(row) != len(cl)
        out.append(row)
    return Cnf.from_clauses(cnf.V, out, cnf.sigma, cnf.name) if changed else cnf


class Oracle:
    """One TurboSAT batch on the CPU: state theta, m, v (fp32, V x Nl) for the
    candidate shard [n0, n0 + Nl) of N global candidates."""

    def __init__(self, cnf, N, seed, cfg: Config | None = None, n0=0, Nl=None, init=True):
        cnf = binary_problem_matrix(cnf)
        self.cnf = cnf
        self.N = int(N)
        self.n0 = int(n0)
        self.Nl = self.N if Nl is None else int(Nl)
        self.seed = int(seed)
        self.cfg = cfg or Config()
        self.K = cnf.K
        self.t = 0
        lits = np.abs(cnf.lits.astype(np.int64)) - 1
        self.occ = np.bincount(lits, minlength=cnf.V).astype(np.int32)
        if init:
            if self.cfg.state_fp64:
                V, Nl = cnf.V, self.Nl
                self.theta = np.empty((V, Nl), np.float64)
                self.m = np.empty((V, Nl), np.float64)
                self.v = np.empty((V, Nl), np.float64)
                lib().or_init64(V, self.n0, Nl, self.seed, _p(self.theta), _p(self.m), _p(self.v))
            else:
                self.theta, self.m, self.v = init_theta(cnf.V, self.N, self.seed, self.n0, self.Nl)
        self.comm = LocalComm()

    @property
    def per_shard(self):
        """normalize = 2 (variant f2): Eq. 5 over this shard's Nl candidates
        only; row sums, J and the J scale's maxima stay local, only the
        selection and the loss are global (each shard is an independent
        instance)."""
        return self.cfg.normalize == 2

    @property
    def Nnorm(self):
        return self.Nl if self.per_shard else self.N

    def set_state(self, theta, m, v, t):
        dt = np.float64 if self.cfg.state_fp64 else np.float32
        self.theta = np.ascontiguousarray(theta, dt).copy()
        self.m = np.ascontiguousarray(m, dt).copy()
        self.v = np.ascontiguousarray(v, dt).copy()
        self.t = int(t)

    def row_stats(self):
        V = self.cnf.V
        Q = np.empty(V, np.int64)
        L = lib()
        if self.cfg.state_fp64:                   # R30: 128-bit row sums at 2^-64 (single shard)
            assert not isinstance(self.comm, object) or isinstance(self.comm, LocalComm) or self.per_shard, \
                "fp64 state: one shard (or per-shard normalisation)"
            Qlo = np.empty(V, np.uint64)
            bad = L.or_row_sums64(V, self.Nl, _p(self.theta), _p(Q), _p(Qlo), int(self.cfg.normalize == 3))
            assert bad == 0, "row-sum bound |theta| < 2^14 (R30)"
            mu = np.empty(V); d = np.empty(V); rho = np.empty(V); guard = np.empty(V, np.uint8)
            L.or_row_finish64(V, self.Nnorm, _p(Q), _p(Qlo), self.cfg.normalize, self.cfg.eps_norm, _p(mu), _p(d),
                              _p(rho), _p(guard))
            self.Qlo = Qlo
            return Q, mu, d, rho, guard
        (L.or_row_sums_abs if self.cfg.normalize == 3 else L.or_row_sums)(V, self.Nl, _p(self.theta), _p(Q))
        if not self.per_shard:
            Q = self.comm.sum_i64(Q)
        thmax_local = float(np.abs(self.theta).max()) if self.theta.size else 0.0
        assert self.N * thmax_local < 2.0 ** 30, "row-sum fixed-point bound (R10)"
        mu = np.empty(V); d = np.empty(V); rho = np.empty(V); guard = np.empty(V, np.uint8)
        L.or_row_finish(V, self.Nnorm, _p(Q), self.cfg.normalize, self.cfg.eps_norm, _p(mu), _p(d), _p(rho),
                        _p(guard))
        return Q, mu, d, rho, guard

    def step(self) -> StepOut:
        cnf, cfg, L = self.cnf, self.cfg, lib()
        V, Nl, K = cnf.V, self.Nl, self.K
        t = self.t
        # Eq. 5 normalisation statistics and Eq. 2 binarisation
        Q, mu, d, rho, guard = self.row_stats()
        b = np.empty((V, Nl), np.uint8)
        f64 = bool(cfg.state_fp64)
        (L.or_binarize64 if f64 else L.or_binarize)(V, Nl, _p(self.theta), _p(d), _p(b))
        # Eq. 1 and §3.1.4
        R = clause_eval(cnf, b)
        h = histogram(R, K)
        unsat = h[:, 0].copy()
        # Eq. 4 / Eq. 3
        S, g, rmin = smoothmin(h, tau_at(t, cfg))
        g32 = g.astype(np.float32)                 # R26: rounded once to fp32
        Sall = self.comm.gather_f64(S)
        loss = -float(sum(float(x) for x in Sall))
        if f64:                                    # R30: the g table, G and J terms stay fp64
            gmax = L.or_gmax64(Nl, K, _p(np.ascontiguousarray(g)), _p(rmin))
            thmax = L.or_abs_max64(self.theta.size, _p(self.theta))
        else:
            gmax = L.or_gmax(Nl, K, _p(g32), _p(rmin))
            thmax = L.or_abs_max(self.theta.size, _p(self.theta))
        if not self.per_shard:
            gmax, thmax = self.comm.max(gmax), self.comm.max(thmax)
        # STE backward and Eq. 5 Jacobian
        I = np.empty(V, np.int64); s = np.empty(V, np.int32); valid = np.empty(V, np.uint8)
        if f64:
            G = np.empty((V, Nl), np.float64)
            L.or_backward64(V, cnf.C, _p(cnf.clause_ptr), _p(cnf.lits), Nl, K, _p(np.ascontiguousarray(R)),
                            _p(np.ascontiguousarray(g)), _p(G))
            L.or_jacobian_partial64(V, Nl, _p(G), _p(self.theta), _p(self.occ), self.Nnorm, gmax, thmax, _p(I),
                                    _p(s), _p(valid))
        else:
            G = backward(cnf, R, g32)                     # fp32 values (R27)
            L.or_jacobian_partial(V, Nl, _p(G), _p(self.theta), _p(self.occ), self.Nnorm, gmax, thmax, _p(I), _p(s),
                                  _p(valid))
        if not self.per_shard:
            I = self.comm.sum_i64(I)
        J = np.empty(V); cv = np.empty(V)
        L.or_jacobian_finish(V, self.Nnorm, _p(I), _p(s), _p(valid), _p(rho), _p(guard), cfg.normalize, _p(J),
                             _p(cv))
        grad = np.empty((V, Nl), np.float64 if f64 else np.float32)
        if f64:
            L.or_grad64(V, Nl, _p(G), _p(rho), _p(cv), _p(self.theta), int(cfg.normalize == 3), _p(grad))
        elif cfg.normalize == 3:
            L.or_grad_mag(V, Nl, _p(G), _p(rho), _p(cv), _p(self.theta), _p(grad))
        else:
            L.or_grad(V, Nl, _p(G), _p(rho), _p(cv), _p(grad))
        # selection (§4.2): best = argmin (unsat, n)
        j = int(np.lexsort((np.arange(Nl), unsat))[0]) if Nl else 0
        key = (int(unsat[j]), self.n0 + j)
        best_unsat, best_idx = self.comm.min_key(key)
        # AdamW + LR schedule (§4.1)
        lr = lr_at(t, cfg)
        reset, bstep = adam_step(t, cfg)
        if reset:
            self.m[:] = 0.0
            self.v[:] = 0.0
        (L.or_adamw64 if f64 else L.or_adamw)(V, self.n0, Nl, _p(self.theta), _p(self.m), _p(self.v), _p(grad), t,
                                               bstep, lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay,
                                               cfg.noise_sigma, self.seed)
        self.t = t + 1
        return StepOut(t=t, bits=b, R=R, h=h, unsat=unsat, S=S, g=g, g32=g32, loss=loss, G=G, grad=grad,
                       J=J, d=d, gmax=gmax, thmax=thmax, best_unsat=best_unsat, best_idx=best_idx,
                       lr=lr, extra=dict(Q=Q, mu=mu, rho=rho, guard=guard, cv=cv, rmin=rmin, I=I, s=s))


def step_sampled(cnf, theta, m, v, t, rows, cfg: Config | None = None):
    """One iteration at full size, for a sample of variable rows (test only).

    Same arithmetic as Oracle.step, organised for large instances: row
    statistics and bits for all variables, the histogram streamed clause by
    clause (no C x N matrix), the g table for all candidates, then the
    backward / Jacobian / AdamW only for `rows`.  theta, m, v are the full
    (V x N) state; returns (unsat, g32, S, loss, theta1, m1, v1) with the last
    three for the sampled rows only."""
    cfg = cfg or Config()
    cnf = binary_problem_matrix(cnf)
    L = lib()
    V, N = theta.shape
    K = cnf.K
    Q = np.empty(V, np.int64)
    (L.or_row_sums_abs if cfg.normalize == 3 else L.or_row_sums)(V, N, _p(theta), _p(Q))
    mu = np.empty(V); d = np.empty(V); rho = np.empty(V); guard = np.empty(V, np.uint8)
    L.or_row_finish(V, N, _p(Q), cfg.normalize, cfg.eps_norm, _p(mu), _p(d), _p(rho), _p(guard))
    b = np.empty((V, N), np.uint8)
    L.or_binarize(V, N, _p(theta), _p(d), _p(b))
    h = np.empty((N, K + 1), np.int32)
    rowbuf = np.empty(N, np.uint8)
    L.or_hist_stream(cnf.C, _p(cnf.clause_ptr), _p(cnf.lits), N, K, _p(b), _p(h), _p(rowbuf))
    S, g, rmin = smoothmin(h, tau_at(t, cfg))
    g32 = g.astype(np.float32)
    loss = -float(sum(float(x) for x in S))
    gmax = L.or_gmax(N, K, _p(g32), _p(rmin))
    thmax = L.or_abs_max(theta.size, _p(theta))
    rows = np.ascontiguousarray(rows, np.int32)
    nr = len(rows)
    G = np.empty((nr, N), np.float64)
    cnt = np.empty((N, K + 1), np.int32)
    L.or_backward_rows(cnf.C, _p(cnf.clause_ptr), _p(cnf.lits), N, K, _p(b), _p(np.ascontiguousarray(g32)),
                       _p(rows), nr, _p(G), _p(cnt), _p(rowbuf))
    occ = np.bincount(np.abs(cnf.lits.astype(np.int64)) - 1, minlength=V).astype(np.int32)[rows]
    th = np.ascontiguousarray(theta[rows]); mm = np.ascontiguousarray(m[rows]); vv = np.ascontiguousarray(v[rows])
    I = np.empty(nr, np.int64); s = np.empty(nr, np.int32); valid = np.empty(nr, np.uint8)
    L.or_jacobian_partial(nr, N, _p(G), _p(th), _p(np.ascontiguousarray(occ)), N, gmax, thmax, _p(I), _p(s), _p(valid))
    J = np.empty(nr); cv = np.empty(nr)
    rho_r = np.ascontiguousarray(rho[rows]); guard_r = np.ascontiguousarray(guard[rows])
    L.or_jacobian_finish(nr, N, _p(I), _p(s), _p(valid), _p(rho_r), _p(guard_r), cfg.normalize, _p(J), _p(cv))
    grad = np.empty((nr, N), np.float32)
    if cfg.normalize == 3:
        L.or_grad_mag(nr, N, _p(G), _p(rho_r), _p(cv), _p(th), _p(grad))
    else:
        L.or_grad(nr, N, _p(G), _p(rho_r), _p(cv), _p(grad))
    lr = lr_at(t, cfg)
    # noise is keyed by the variable index: only sigma = 0 here
    assert cfg.noise_sigma == 0.0
    reset, bstep = adam_step(t, cfg)
    if reset:
        mm[:] = 0.0
        vv[:] = 0.0
    L.or_adamw(nr, 0, N, _p(th), _p(mm), _p(vv), _p(grad), t, bstep, lr, cfg.beta1, cfg.beta2, cfg.eps,
               cfg.weight_decay, 0.0, 0)
    return h[:, 0].copy(), g32, S, loss, th, mm, vv
