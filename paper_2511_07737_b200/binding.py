"""Thin ctypes binding of libturbosat (include/turbosat.h): argument marshalling
only.  Every step of the path runs in the library's CUDA kernels; PyTorch only
provides device memory (the workspace tensor) and the CUDA stream.  There is no
CPU fallback: if the shared library is missing or no CUDA device is present the
calls fail loudly.
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSAT_LIB") or os.path.join(HERE, "libturbosat.so")
PEER_HANDLE_BYTES = 64          # TSAT_PEER_HANDLE_BYTES

TSAT_STATUS = {
    0: "TSAT_OK", 1: "TSAT_E_ARG", 2: "TSAT_E_PARSE", 3: "TSAT_E_RANGE", 4: "TSAT_E_STATE",
    5: "TSAT_E_OOM", 6: "TSAT_E_CUDA", 7: "TSAT_E_NCCL", 8: "TSAT_E_UNSUPPORTED",
}


class TsatError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        self.name = TSAT_STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


class tsat_config(ct.Structure):
    _fields_ = [("tau", ct.c_double), ("normalize", ct.c_int32), ("beta1", ct.c_double), ("beta2", ct.c_double),
                ("eps", ct.c_double), ("weight_decay", ct.c_double), ("lr0", ct.c_double), ("lr_min", ct.c_double),
                ("decay_factor", ct.c_double), ("decay_every", ct.c_int32), ("restart_every", ct.c_int32),
                ("noise_sigma", ct.c_double), ("eps_norm", ct.c_double), ("reset_moments_on_restart", ct.c_int32),
                ("tau_final", ct.c_double), ("clause_eval", ct.c_int32), ("state_fp64", ct.c_int32)]


class tsat_cnf_info(ct.Structure):
    _fields_ = [("V", ct.c_int32), ("C", ct.c_int64), ("nnz", ct.c_int64), ("K", ct.c_int32),
                ("header_C", ct.c_int64), ("n_warnings", ct.c_int64), ("n_tautologies", ct.c_int64),
                ("n_duplicates", ct.c_int64), ("has_empty", ct.c_int32), ("n_hub_rows", ct.c_int32)]


class tsat_step_info(ct.Structure):
    _fields_ = [("t", ct.c_int64), ("best_unsat", ct.c_int32), ("best_idx", ct.c_int64), ("solved", ct.c_int32),
                ("solved_step", ct.c_int64), ("solved_idx", ct.c_int64), ("loss", ct.c_double)]


class tsat_cdcl_result(ct.Structure):
    _fields_ = [("status", ct.c_int32), ("winner", ct.c_int32), ("seconds", ct.c_double), ("conflicts", ct.c_int64),
                ("decisions", ct.c_int64), ("propagations", ct.c_int64), ("failed_seeds", ct.c_int32),
                ("threads", ct.c_int32)]


class tsat_partial(ct.Structure):
    _fields_ = [("candidate", ct.c_int64), ("unsat", ct.c_int32), ("k", ct.c_int32),
                ("lits", ct.POINTER(ct.c_int32)), ("abs_grad", ct.POINTER(ct.c_float))]


P = ct.c_void_p
_SIGS = {
    "tsat_config_default": (ct.c_int, [ct.POINTER(tsat_config)]),
    "tsat_parse_dimacs": (ct.c_int, [ct.c_char_p, ct.c_size_t, ct.POINTER(tsat_cnf_info)]),
    "tsat_status_string": (ct.c_char_p, [ct.c_int]),
    "tsat_nccl_unique_id": (ct.c_int, [P, ct.c_size_t]),
    "tsat_create": (ct.c_int, [ct.POINTER(P), ct.c_int, P, P, ct.c_int, ct.c_int]),
    "tsat_create_peer": (ct.c_int, [ct.POINTER(P), ct.c_int, P, ct.c_int, ct.c_int]),
    "tsat_peer_handle": (ct.c_int, [P, P, ct.c_size_t]),
    "tsat_peer_open": (ct.c_int, [P, P, ct.c_size_t]),
    "tsat_load_dimacs": (ct.c_int, [P, ct.c_char_p, ct.c_size_t, ct.POINTER(tsat_cnf_info)]),
    "tsat_load_clauses": (ct.c_int, [P, ct.c_int32, ct.c_int64, P, P, ct.POINTER(tsat_cnf_info)]),
    "tsat_workspace_bytes": (ct.c_int, [P, ct.c_int64, ct.POINTER(ct.c_size_t)]),
    "tsat_init_batch": (ct.c_int, [P, ct.c_int64, ct.c_uint64, ct.POINTER(tsat_config), P, ct.c_size_t]),
    "tsat_step": (ct.c_int, [P, ct.c_int32, ct.POINTER(tsat_step_info)]),
    "tsat_get_info": (ct.c_int, [P, ct.POINTER(tsat_step_info)]),
    "tsat_query_unsat_async": (ct.c_int, [P, P, ct.c_size_t, ct.POINTER(ct.c_int64)]),
    "tsat_sync": (ct.c_int, [P]),
    "tsat_query_unsat": (ct.c_int, [P, P, ct.c_size_t, ct.POINTER(ct.c_int64)]),
    "tsat_export_best": (ct.c_int, [P, ct.c_int32, ct.c_int32, ct.POINTER(tsat_partial)]),
    "tsat_export_k": (ct.c_int, [P, ct.c_int32, ct.POINTER(ct.c_int32)]),
    "tsat_merge_keys": (ct.c_int, [P, ct.c_size_t, ct.c_int32, P]),
    "tsat_cdcl_solve": (ct.c_int, [ct.c_int32, ct.c_int64, P, P, ct.c_int32, P, ct.c_int64, ct.c_uint64, P,
                                   ct.POINTER(tsat_cdcl_result)]),
    "tsat_cdcl_portfolio": (ct.c_int, [ct.c_int32, ct.c_int64, P, P, ct.c_int32, ct.c_int32, P, ct.c_int32,
                                       ct.c_int32, ct.c_double, P, ct.POINTER(tsat_cdcl_result)]),
    "tsat_gen_planted": (ct.c_int, [ct.c_int32, ct.c_int64, ct.c_int32, ct.c_uint64, ct.c_int32, P, P, P]),
    "tsat_gen_industrial": (ct.c_int, [ct.c_int32, ct.c_int64, ct.c_uint64, ct.c_double, ct.c_int32, P, P, P,
                                       ct.c_int64, P]),
    "tsat_write_dimacs": (ct.c_int, [ct.c_int32, ct.c_int64, P, P, P, P, ct.c_size_t, ct.POINTER(ct.c_size_t)]),
    "tsat_verify_model": (ct.c_int, [ct.c_int32, ct.c_int64, P, P, P, ct.POINTER(ct.c_int64)]),
    "tsat_lr_at": (ct.c_int, [ct.POINTER(tsat_config), ct.c_int64, ct.POINTER(ct.c_double)]),
    "tsat_export_model": (ct.c_int, [P, ct.c_int64, P]),
    "tsat_get_solution": (ct.c_int, [P, P, ct.POINTER(ct.c_int64), ct.POINTER(ct.c_int64)]),
    "tsat_get_state": (ct.c_int, [P, P, P, P, ct.c_size_t, ct.POINTER(ct.c_int64)]),
    "tsat_set_state": (ct.c_int, [P, P, P, P, ct.c_size_t, ct.c_int64]),
    "tsat_get_state64": (ct.c_int, [P, P, P, P, ct.c_size_t, ct.POINTER(ct.c_int64)]),
    "tsat_set_state64": (ct.c_int, [P, P, P, P, ct.c_size_t, ct.c_int64]),
    "tsat_debug_copy": (ct.c_int, [P, ct.c_int32, P, ct.c_size_t]),
    "tsat_get_rows": (ct.c_int, [P, P, ct.c_int32, P, P, P, ct.c_size_t]),
    "tsat_set_profiling": (ct.c_int, [P, ct.c_int32]),
    "tsat_kernel_times": (ct.c_int, [P, P, ct.POINTER(ct.c_int64)]),
    "tsat_kernels_per_step": (ct.c_int, [P, ct.POINTER(ct.c_int32)]),
    "tsat_update_geometry": (ct.c_int, [P, P, ct.c_int32]),
    "tsat_error_string": (ct.c_char_p, [P]),
    "tsat_destroy": (None, [P]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libturbosat.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not found: build it with `python -m paper_2511_07737_b200.build` "
                              "(there is no CPU fallback)")
        lib = ct.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:          # an older library build (A/B variants): that entry point is absent
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return ct.c_void_p(a.ctypes.data)


def config_default() -> tsat_config:
    c = tsat_config()
    load_library().tsat_config_default(ct.byref(c))
    return c


def parse_dimacs(text: bytes) -> tsat_cnf_info:
    """tsat_parse_dimacs: host-only DIMACS validation."""
    info = tsat_cnf_info()
    s = load_library().tsat_parse_dimacs(text, len(text), ct.byref(info))
    if s:
        raise TsatError(s, "DIMACS rejected")
    return info


def gen_planted(V: int, C: int, k: int = 3, seed: int = 1, hidden: int = 1):
    """tsat_gen_planted (host only): (clause_ptr int64[C+1], lits int32[C*k], sigma uint8[V])."""
    ptr = np.zeros(C + 1, np.int64)
    lits = np.zeros(max(C * k, 1), np.int32)
    sigma = np.zeros(V, np.uint8)
    st = load_library().tsat_gen_planted(int(V), int(C), int(k), int(seed) & (2**64 - 1), int(hidden), _ptr(ptr),
                                         _ptr(lits), _ptr(sigma))
    if st:
        raise TsatError(st, "tsat_gen_planted")
    return ptr, lits[:C * k], sigma


def gen_industrial(V: int, C: int, seed: int = 1, alpha: float = 0.82, len_probs=None):
    """tsat_gen_industrial (host only); len_probs maps clause length -> probability
    (default SURVEY §8(d): {2:.40, 3:.30, 4:.12, 5:.08, 6:.06, 7:.04})."""
    lp = len_probs or {2: .40, 3: .30, 4: .12, 5: .08, 6: .06, 7: .04}
    kmax = max(lp)
    probs = np.zeros(kmax + 1, np.float64)
    for k, p in lp.items():
        probs[k] = p
    ptr = np.zeros(C + 1, np.int64)
    lits = np.zeros(max(C * kmax, 1), np.int32)
    sigma = np.zeros(V, np.uint8)
    st = load_library().tsat_gen_industrial(int(V), int(C), int(seed) & (2**64 - 1), float(alpha), kmax, _ptr(probs),
                                            _ptr(ptr), _ptr(lits), lits.size, _ptr(sigma))
    if st:
        raise TsatError(st, "tsat_gen_industrial")
    return ptr, lits[:ptr[-1]].copy(), sigma


def write_dimacs(V: int, clause_ptr, lits, sigma=None) -> bytes:
    """tsat_write_dimacs (host only)."""
    ptr = np.ascontiguousarray(clause_ptr, np.int64)
    lt = np.ascontiguousarray(lits, np.int32)
    sg = None if sigma is None else np.ascontiguousarray(sigma, np.uint8)
    n = ct.c_size_t()
    C = len(ptr) - 1
    L = load_library()
    args = (int(V), C, _ptr(ptr), _ptr(lt) if lt.size else None, _ptr(sg) if sg is not None else None)
    st = L.tsat_write_dimacs(*args, None, 0, ct.byref(n))
    if st:
        raise TsatError(st, "tsat_write_dimacs")
    buf = ct.create_string_buffer(n.value)
    st = L.tsat_write_dimacs(*args, buf, n.value, ct.byref(n))
    if st:
        raise TsatError(st, "tsat_write_dimacs")
    return buf.raw[:n.value]


def verify_model(V: int, clause_ptr, lits, model) -> int:
    """tsat_verify_model (host only): clauses the 0/1 assignment leaves unsatisfied."""
    ptr = np.ascontiguousarray(clause_ptr, np.int64)
    lt = np.ascontiguousarray(lits, np.int32)
    m = np.ascontiguousarray(model, np.uint8)
    out = ct.c_int64()
    st = load_library().tsat_verify_model(int(V), len(ptr) - 1, _ptr(ptr), _ptr(lt) if lt.size else None, _ptr(m),
                                          ct.byref(out))
    if st:
        raise TsatError(st, "tsat_verify_model")
    return int(out.value)


def cdcl_solve(cnf, assumptions=(), conflict_limit: int = 0, seed: int = 0):
    """tsat_cdcl_solve (host only): one CDCL run under assumed DIMACS literals.
    Returns (result, model or None)."""
    ptr = np.ascontiguousarray(cnf.clause_ptr, np.int64)
    lits = np.ascontiguousarray(cnf.lits, np.int32)
    a = np.ascontiguousarray(np.asarray(assumptions, np.int32).reshape(-1))
    model = np.zeros(cnf.V, np.uint8)
    res = tsat_cdcl_result()
    st = load_library().tsat_cdcl_solve(cnf.V, cnf.C, _ptr(ptr), _ptr(lits), a.size, _ptr(a) if a.size else None,
                                        int(conflict_limit), int(seed), _ptr(model), ct.byref(res))
    if st:
        raise TsatError(st, "tsat_cdcl_solve")
    return res, (model if res.status == 10 else None)


def cdcl_portfolio(cnf, seeds, threads: int, unseeded: bool = True, time_limit_s: float = 60.0):
    """tsat_cdcl_portfolio (host only): seeds = M x k signed DIMACS literals
    (tsat_export_best's lits, best candidate first).  Returns (result, model or None)."""
    ptr = np.ascontiguousarray(cnf.clause_ptr, np.int64)
    lits = np.ascontiguousarray(cnf.lits, np.int32)
    sd = np.ascontiguousarray(np.asarray(seeds, np.int32))
    M, k = (sd.shape if sd.ndim == 2 else (0, 0))
    model = np.zeros(cnf.V, np.uint8)
    res = tsat_cdcl_result()
    st = load_library().tsat_cdcl_portfolio(cnf.V, cnf.C, _ptr(ptr), _ptr(lits), M, k, _ptr(sd) if sd.size else None,
                                            int(threads), int(bool(unseeded)), float(time_limit_s), _ptr(model),
                                            ct.byref(res))
    if st:
        raise TsatError(st, "tsat_cdcl_portfolio")
    return res, (model if res.status == 10 else None)


def lr_at(cfg: tsat_config, t: int) -> float:
    """tsat_lr_at (host only): the learning rate of iteration t."""
    out = ct.c_double()
    st = load_library().tsat_lr_at(ct.byref(cfg), int(t), ct.byref(out))
    if st:
        raise TsatError(st, "tsat_lr_at")
    return out.value


def nccl_unique_id() -> bytes:
    """tsat_nccl_unique_id: 128 bytes, to be broadcast to every rank."""
    buf = ct.create_string_buffer(128)
    s = load_library().tsat_nccl_unique_id(buf, 128)
    if s:
        raise TsatError(s, "ncclGetUniqueId failed")
    return buf.raw


def merge_keys(keys: np.ndarray, M: int) -> np.ndarray:
    """tsat_merge_keys (host only): the M smallest (unsat << 32 | index) keys."""
    k = np.ascontiguousarray(keys, np.uint64)
    out = np.empty(M, np.uint64)
    s = load_library().tsat_merge_keys(_ptr(k), k.size, int(M), _ptr(out))
    if s:
        raise TsatError(s, "tsat_merge_keys")
    return out


@dataclass
class StepInfo:
    t: int
    best_unsat: int
    best_idx: int
    solved: bool
    solved_step: int
    solved_idx: int
    loss: float


class Solver:
    """One TurboSAT batch on one CUDA device (rank `rank` of `world`).

    Mirrors the C-ABI: load_dimacs / load_clauses -> init_batch -> step(k) ->
    query_unsat / export_best / export_model / get_solution; get_state /
    set_state for checkpoint-resume."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1, nccl_unique_id: bytes | None = None,
                 peer: bool = False):
        """world > 1 (or a unique id with world == 1): candidate-sharded path;
        every rank must construct its Solver concurrently with the same id
        (see Solver.distributed).  peer=True: the peer-exchange path
        (tsat_create_peer; connect with peer_handle / peer_open after loading
        the CNF, see Solver.connect_peers)."""
        import torch
        self._torch = torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2511_07737_b200 needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = device
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ct.c_void_p()
        if peer:
            self._check(self.lib.tsat_create_peer(ct.byref(h), device, ct.c_void_p(self.stream.cuda_stream), rank, world),
                        None)
        else:
            uid = ct.c_char_p(nccl_unique_id) if nccl_unique_id is not None else None
            self._check(self.lib.tsat_create(ct.byref(h), device, ct.c_void_p(self.stream.cuda_stream), uid, rank, world),
                        None)
        self.peer = peer
        self.h = h
        self.ws = None
        self.V = self.C = self.N = self.N_local = 0
        self.rank, self.world = rank, world
        self.n0 = 0
        self.info = None

    @classmethod
    def distributed(cls, device: int, rank: int, world: int, stream=None, group=None):
        """Sharded solver over a torch.distributed group: rank 0 makes the NCCL
        unique id, every rank receives it (broadcast_object_list) and joins."""
        import torch.distributed as dist
        obj = [nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(device, stream=stream, rank=rank, world=world, nccl_unique_id=obj[0])

    # -- peer-exchange path
    def peer_handle(self) -> bytes:
        """This rank's exchange-buffer IPC handle (after load_*)."""
        buf = ct.create_string_buffer(PEER_HANDLE_BYTES)
        self._check(self.lib.tsat_peer_handle(self.h, buf, PEER_HANDLE_BYTES))
        return buf.raw

    def peer_open(self, handles) -> None:
        """Map every rank's exchange buffer (handles in rank order)."""
        blob = b"".join(handles)
        self._check(self.lib.tsat_peer_open(self.h, blob, len(blob)))

    def connect_peers(self, group=None) -> None:
        """All-gather the handles over torch.distributed (any backend, e.g.
        gloo) and map them; call on every rank after load_*."""
        import torch.distributed as dist
        hs = [None] * self.world
        mine = self.peer_handle()
        if self.world > 1:
            dist.all_gather_object(hs, mine, group=group)
        else:
            hs = [mine]
        self.peer_open(hs)

    # -- helpers
    def _check(self, s, h="self"):
        if s:
            msg = ""
            hh = self.h if h == "self" else h
            if hh is not None:
                msg = (self.lib.tsat_error_string(hh) or b"").decode()
            raise TsatError(s, msg)

    def close(self):
        if getattr(self, "h", None):
            self.lib.tsat_destroy(self.h)
            self.h = None
            self.ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- C-ABI mirrors
    def load_dimacs(self, text: bytes) -> tsat_cnf_info:
        info = tsat_cnf_info()
        self._check(self.lib.tsat_load_dimacs(self.h, text, len(text), ct.byref(info)))
        self.V, self.C, self.info = info.V, info.C, info
        return info

    def load_clauses(self, V: int, clause_ptr: np.ndarray, lits: np.ndarray) -> tsat_cnf_info:
        cp = np.ascontiguousarray(clause_ptr, np.int64)
        li = np.ascontiguousarray(lits, np.int32)
        info = tsat_cnf_info()
        self._check(self.lib.tsat_load_clauses(self.h, int(V), len(cp) - 1, _ptr(cp), _ptr(li), ct.byref(info)))
        self.V, self.C, self.info = info.V, info.C, info
        return info

    def load_cnf(self, cnf) -> tsat_cnf_info:
        return self.load_clauses(cnf.V, cnf.clause_ptr, cnf.lits)

    def workspace_bytes(self, N_global: int) -> int:
        b = ct.c_size_t()
        self._check(self.lib.tsat_workspace_bytes(self.h, int(N_global), ct.byref(b)))
        return b.value

    def init_batch(self, N_global: int, seed: int, cfg: tsat_config | None = None, **overrides):
        torch = self._torch
        if cfg is None:
            cfg = config_default()
        for k, v in overrides.items():
            setattr(cfg, k, v)
        nbytes = self.workspace_bytes(N_global)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        self._check(self.lib.tsat_init_batch(self.h, int(N_global), int(seed) & (2**64 - 1), ct.byref(cfg),
                                             ct.c_void_p(self.ws.data_ptr()), nbytes))
        self.N = int(N_global)
        self.fp64 = bool(cfg.state_fp64)
        self.N_local = self.N // self.world
        self.n0 = self.rank * self.N_local
        return self

    def step(self, k: int = 1, wait: bool = True) -> StepInfo | None:
        if not wait:
            self._check(self.lib.tsat_step(self.h, int(k), None))
            return None
        si = tsat_step_info()
        self._check(self.lib.tsat_step(self.h, int(k), ct.byref(si)))
        return StepInfo(si.t, si.best_unsat, si.best_idx, bool(si.solved), si.solved_step, si.solved_idx, si.loss)

    def get_info(self) -> StepInfo:
        si = tsat_step_info()
        self._check(self.lib.tsat_get_info(self.h, ct.byref(si)))
        return StepInfo(si.t, si.best_unsat, si.best_idx, bool(si.solved), si.solved_step, si.solved_idx, si.loss)

    def query_unsat(self, out: np.ndarray | None = None) -> np.ndarray:
        n = self.N_local_count()
        if out is None:
            out = np.empty(n, np.int32)
        if out.dtype != np.int32 or out.shape != (n,) or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a contiguous int32 array of shape ({n},)")
        first = ct.c_int64()
        self._check(self.lib.tsat_query_unsat(self.h, _ptr(out), out.size, ct.byref(first)))
        self.n0 = first.value
        return out

    def query_unsat_async(self, out_ptr: int, n: int | None = None) -> None:
        """Enqueue the unsat-count copy into PINNED host memory at out_ptr
        (n = N_local int32); valid after sync() or another blocking call."""
        first = ct.c_int64()
        n = self.N_local_count() if n is None else int(n)
        self._check(self.lib.tsat_query_unsat_async(self.h, ct.c_void_p(int(out_ptr)), n, ct.byref(first)))
        self.n0 = first.value

    def sync(self) -> None:
        self._check(self.lib.tsat_sync(self.h))

    def N_local_count(self) -> int:
        return self.N // self.world

    def export_best(self, M: int, k: int = 0):
        """tsat_export_best: the M best candidates over all ranks (a collective
        call when world > 1), each with its k most confident literals; k <= 0
        lets the library apply the paper's rule (buffers sized for k = V)."""
        kk = ct.c_int32()
        self._check(self.lib.tsat_export_k(self.h, int(k), ct.byref(kk)))
        kk = kk.value
        bufs = []
        arr = (tsat_partial * M)()
        for i in range(M):
            lits = np.zeros(kk, np.int32)
            g = np.zeros(kk, np.float32)
            bufs.append((lits, g))
            arr[i].lits = lits.ctypes.data_as(ct.POINTER(ct.c_int32))
            arr[i].abs_grad = g.ctypes.data_as(ct.POINTER(ct.c_float))
        self._check(self.lib.tsat_export_best(self.h, int(M), int(k), arr))
        return [dict(candidate=arr[i].candidate, unsat=arr[i].unsat, lits=bufs[i][0][:arr[i].k].copy(),
                     abs_grad=bufs[i][1][:arr[i].k].copy()) for i in range(M)]

    def export_model(self, idx: int) -> np.ndarray:
        out = np.empty(self.V, np.uint8)
        self._check(self.lib.tsat_export_model(self.h, int(idx), _ptr(out)))
        return out

    def get_solution(self):
        out = np.empty(self.V, np.uint8)
        idx, st = ct.c_int64(), ct.c_int64()
        s = self.lib.tsat_get_solution(self.h, _ptr(out), ct.byref(idx), ct.byref(st))
        if s == 4:
            return None
        self._check(s)
        return out, idx.value, st.value

    def get_state(self):
        """(theta, m, v, t): float32 arrays, or float64 for a batch with state_fp64 = 1."""
        n = self.N_local_count()
        f64 = getattr(self, "fp64", False)
        th = np.empty((self.V, n), np.float64 if f64 else np.float32)
        m = np.empty_like(th)
        v = np.empty_like(th)
        t = ct.c_int64()
        fn = self.lib.tsat_get_state64 if f64 else self.lib.tsat_get_state
        self._check(fn(self.h, _ptr(th), _ptr(m), _ptr(v), th.size, ct.byref(t)))
        return th, m, v, t.value

    def set_state(self, theta, m, v, t: int):
        shape = (self.V, self.N_local_count())
        f64 = getattr(self, "fp64", False)
        dt = np.float64 if f64 else np.float32
        arrs = []
        for name, x in (("theta", theta), ("m", m), ("v", v)):
            x = np.asarray(x)
            if x.dtype != dt or x.shape != shape:
                raise ValueError(f"{name} must be {dt.__name__} of shape {shape} (got {x.dtype} {x.shape})")
            arrs.append(np.ascontiguousarray(x))
        th, mm, vv = arrs
        fn = self.lib.tsat_set_state64 if f64 else self.lib.tsat_set_state
        self._check(fn(self.h, _ptr(th), _ptr(mm), _ptr(vv), th.size, int(t)))

    def get_rows(self, rows):
        r = np.ascontiguousarray(rows, np.int32)
        n = self.N_local_count()
        th = np.empty((len(r), n), np.float32)
        m = np.empty_like(th)
        v = np.empty_like(th)
        self._check(self.lib.tsat_get_rows(self.h, _ptr(r), len(r), _ptr(th), _ptr(m), _ptr(v), n))
        return th, m, v

    def debug(self, which: int, dtype, shape) -> np.ndarray:
        out = np.empty(shape, dtype)
        self._check(self.lib.tsat_debug_copy(self.h, int(which), _ptr(out), out.nbytes))
        return out

    def set_profiling(self, on: bool):
        self._check(self.lib.tsat_set_profiling(self.h, 1 if on else 0))

    def kernel_times(self):
        ms = np.zeros(5, np.float64)
        st = ct.c_int64()
        self._check(self.lib.tsat_kernel_times(self.h, _ptr(ms), ct.byref(st)))
        return ms, st.value

    def update_geometry(self) -> dict:
        g = np.zeros(8, np.int32)
        self._check(self.lib.tsat_update_geometry(self.h, _ptr(g), 8))
        keys = ("GT", "groups", "grid", "smem", "slice", "cluster", "rows_per_item", "clause_segments")
        return {k: int(x) for k, x in zip(keys, g)}

    def kernels_per_step(self) -> int:
        n = ct.c_int32()
        self._check(self.lib.tsat_kernels_per_step(self.h, ct.byref(n)))
        return n.value
