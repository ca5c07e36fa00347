"""Seeded synthetic inputs for TurboSAT parity tests and benchmarks.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA
path (``paper_2511_07737_b200/``).  It holds none of the method's arithmetic:
it produces CNF instances (clause arrays / DIMACS text) and, for tests, raw
state arrays.  Every generator is a pure function of its seed (numpy PCG64).

Workload recipes:

* ``planted_ksat``   - planted random k-SAT: sigma uniform; each clause picks k
  distinct variables uniformly; literal signs uniform over the 2^k - 1 sign
  patterns that sigma satisfies.  Paper workloads are SAT-Competition
  satisfiable instances (§5 l.307); planted instances are satisfiable
  by construction, like them.
* ``industrial_cnf`` - "industrial-shaped": clause lengths i.i.d. from
  {2:.40, 3:.30, 4:.12, 5:.08, 6:.06, 7:.04}; variables drawn with probability
  proportional to rank^-0.82 (scale-free structure the paper cites for
  industrial instances, §4.2 l.292) under a random id permutation;
  k distinct variables per clause; signs planted as above.
* ``coloring_cnf``   - planted graph k-colouring (the shape of PAPER.md Table 1's
  ``6g_6color`` family, l.345): variables x_{u,c}; one at-least-one clause of
  length k per node (long clauses: k up to 15), at-most-one pairs
  (-x_{u,c} v -x_{u,d}) and edge conflicts (-x_{u,c} v -x_{w,c}) over a random
  graph properly coloured by a hidden colouring.
* ``fig1_cnf``       - the 4-variable / 5-clause example of PAPER.md Fig. 1/2
  (§3.1, l.45-53, l.84-95) in SPEC.md's reconstruction.
* ``enumeration_theta`` - theta = +-1 from the bits of the candidate index, so
  the N = 2^V candidates enumerate every assignment (brute-force pin).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "Cnf",
    "planted_ksat",
    "industrial_cnf",
    "fig1_cnf",
    "coloring_cnf",
    "literal_split",
    "to_dimacs",
    "enumeration_theta",
    "random_state",
    "CONFIGS",
    "make_config",
]


class Cnf:
    """A CNF instance as flat arrays.

    ``clause_ptr`` (int64, C+1) and ``lits`` (int32, nnz) hold signed 1-based
    DIMACS literals: clause c is ``lits[clause_ptr[c]:clause_ptr[c+1]]``.
    ``sigma`` (uint8, V) is the planted model when known, else None.
    """

    def __init__(self, V, clause_ptr, lits, sigma=None, name=""):
        self.V = int(V)
        self.clause_ptr = np.ascontiguousarray(clause_ptr, dtype=np.int64)
        self.lits = np.ascontiguousarray(lits, dtype=np.int32)
        self.sigma = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.uint8)
        self.name = name

    @property
    def C(self) -> int:
        return len(self.clause_ptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.clause_ptr[-1])

    @property
    def K(self) -> int:
        if self.C == 0:
            return 0
        return int(np.diff(self.clause_ptr).max())

    def clauses(self):
        """List of clauses (lists of signed ints) - for small instances only."""
        p, l = self.clause_ptr, self.lits
        return [l[p[c]:p[c + 1]].tolist() for c in range(self.C)]

    @staticmethod
    def from_clauses(V, clauses, sigma=None, name=""):
        ptr = np.zeros(len(clauses) + 1, dtype=np.int64)
        for i, c in enumerate(clauses):
            ptr[i + 1] = ptr[i] + len(c)
        lits = np.array([x for c in clauses for x in c], dtype=np.int32)
        return Cnf(V, ptr, lits, sigma, name)


def _distinct_rows(rng, draw, rows, k):
    """Draw a (rows, k) int64 matrix with distinct entries per row.

    ``draw(n)`` returns n iid variable ids; rows containing a repeat are
    redrawn until none remain (rejection sampling, so each row is an iid
    draw conditioned on distinctness)."""
    out = draw(rows * k).reshape(rows, k)
    if k == 1:
        return out
    while True:
        s = np.sort(out, axis=1)
        bad = np.nonzero((s[:, 1:] == s[:, :-1]).any(axis=1))[0]
        if bad.size == 0:
            return out
        out[bad] = draw(bad.size * k).reshape(bad.size, k)


def _plant_signs(rng, vars_, sigma, lens=None, hidden=1):
    """Signs uniform over the patterns that sigma satisfies.

    vars_ is (C, kmax) (entries beyond ``lens`` ignored).  For each clause a
    truth pattern t in [1, 2^len - 1] is drawn uniformly; literal i is made
    true under sigma iff bit i of t is set.  hidden=2 ("2-hidden" planting,
    SURVEY §8(f) f2): t in [1, 2^len - 2], so the complement of sigma
    satisfies every clause too and a literal's polarity carries no majority
    signal about sigma (each literal agrees with sigma with probability 1/2)."""
    C, kmax = vars_.shape
    if lens is None:
        lens = np.full(C, kmax, dtype=np.int64)
    npat = (1 << lens) - (1 if hidden == 1 else 2)
    t = np.floor(rng.random(C) * npat).astype(np.int64) + 1
    bits = (t[:, None] >> np.arange(kmax)[None, :]) & 1          # literal true under sigma?
    sv = sigma[vars_].astype(np.int64)                             # sigma value of the variable
    positive = (bits == sv)                                        # positive literal true iff sigma=1
    return np.where(positive, vars_ + 1, -(vars_ + 1)).astype(np.int32)


def planted_ksat(V: int, C: int, k: int = 3, seed: int = 1, hidden: int = 1) -> Cnf:
    """Planted random k-SAT (SURVEY §8(d) 'planted-k-SAT (naive)'); hidden=2:
    2-hidden planting (sigma and its complement both satisfy, k >= 2)."""
    if hidden == 2 and k < 2:
        raise ValueError("2-hidden planting needs k >= 2")
    key = [0x7A7, int(seed), int(V), int(C), int(k)] + ([2] if hidden == 2 else [])
    rng = np.random.default_rng(key)
    sigma = rng.integers(0, 2, size=V, dtype=np.uint8)
    vars_ = _distinct_rows(rng, lambda n: rng.integers(0, V, size=n), C, k)
    lits = _plant_signs(rng, vars_, sigma, hidden=hidden)
    ptr = np.arange(C + 1, dtype=np.int64) * k
    tag = "planted2" if hidden == 2 else "planted"
    return Cnf(V, ptr, lits.reshape(-1), sigma, f"{tag}-{k}sat-V{V}-C{C}-s{seed}")


INDUSTRIAL_LENGTHS = {2: 0.40, 3: 0.30, 4: 0.12, 5: 0.08, 6: 0.06, 7: 0.04}


def industrial_cnf(V: int, C: int, seed: int = 1, alpha: float = 0.82,
                   lengths=INDUSTRIAL_LENGTHS) -> Cnf:
    """Industrial-shaped CNF: mixed lengths, power-law occurrences."""
    rng = np.random.default_rng([0x1D5, int(seed), int(V), int(C)])
    sigma = rng.integers(0, 2, size=V, dtype=np.uint8)
    ks = np.array(sorted(lengths), dtype=np.int64)
    ps = np.array([lengths[x] for x in ks], dtype=np.float64)
    ps /= ps.sum()
    lens = ks[rng.choice(len(ks), size=C, p=ps)]
    w = np.arange(1, V + 1, dtype=np.float64) ** (-alpha)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    perm = rng.permutation(V)

    def draw(n):
        r = np.searchsorted(cdf, rng.random(n), side="right")
        return perm[np.minimum(r, V - 1)]

    kmax = int(lens.max()) if C else 0
    vars_ = np.zeros((C, kmax), dtype=np.int64)
    for k in ks:
        rows = np.nonzero(lens == k)[0]
        if rows.size:
            vars_[rows, :k] = _distinct_rows(rng, draw, rows.size, int(k))
    lits2 = _plant_signs(rng, vars_, sigma, lens)
    mask = np.arange(kmax)[None, :] < lens[:, None]
    ptr = np.zeros(C + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    return Cnf(V, ptr, lits2[mask], sigma, f"industrial-V{V}-C{C}-s{seed}")


def coloring_cnf(nodes: int, colors: int, degree: int = 4, seed: int = 1) -> Cnf:
    """Planted graph colouring CNF: clause lengths 2 and `colors` (K = colors)."""
    rng = np.random.default_rng([0xC010, int(seed), int(nodes), int(colors), int(degree)])
    col = rng.integers(0, colors, size=nodes)
    var = lambda u, c: int(u) * colors + int(c) + 1
    cl = [[var(u, c) for c in range(colors)] for u in range(nodes)]            # at least one colour
    for u in range(nodes):                                                      # at most one colour
        for c in range(colors):
            for d in range(c + 1, colors):
                cl.append([-var(u, c), -var(u, d)])
    m = nodes * degree // 2
    a, b = rng.integers(0, nodes, size=m), rng.integers(0, nodes, size=m)
    for u, w in zip(a, b):
        if u != w and col[u] != col[w]:                                         # edges the hidden colouring respects
            for c in range(colors):
                cl.append([-var(u, c), -var(w, c)])
    sigma = np.zeros(nodes * colors, dtype=np.uint8)
    sigma[np.arange(nodes) * colors + col] = 1
    cnf = Cnf.from_clauses(nodes * colors, cl, name=f"color{colors}-n{nodes}-d{degree}-s{seed}")
    cnf.sigma = sigma
    return cnf


def literal_split(cnf: Cnf) -> Cnf:
    """The 2V-literal-row form of PAPER.md l.191 (A_real is 2V x N): literal
    +v becomes variable v and literal -v becomes variable V + v, both
    positive, so each literal row has its own parameters and its own Eq. 5
    normalisation and nothing keeps the two rows of a variable complementary
    (reading R2 does; this is the alternative the verdict asked to test).
    sigma extends to (sigma, 1 - sigma).  Pure relabelling: no method arithmetic."""
    lits = np.asarray(cnf.lits, np.int64)
    out = np.where(lits > 0, lits, cnf.V - lits).astype(np.int32)        # -v -> V + v (1-based)
    sigma = None if cnf.sigma is None else np.concatenate([cnf.sigma, 1 - cnf.sigma]).astype(np.uint8)
    return Cnf(2 * cnf.V, cnf.clause_ptr.copy(), out, sigma, cnf.name + "-2V")


def fig1_cnf() -> Cnf:
    """PAPER.md Fig. 1/2 example (4 vars, 5 clauses), SPEC.md S:47 reconstruction.

    Paper-pinned facts: clause 2 = (x3 v x4) (l.148); clause 3 = (~x1 v ~x3)
    (implied by l.165-166); clauses 1, 4, 5 are the reconstruction's."""
    return Cnf.from_clauses(4, [[1, 2], [3, 4], [-1, -3], [-2, 4], [1, -4]], name="fig1")


def to_dimacs(cnf: Cnf, comment: str | None = None) -> bytes:
    """Serialise to DIMACS text (planted sigma, if any, in a comment)."""
    out = []
    if comment:
        out.append(f"c {comment}\n")
    if cnf.sigma is not None and cnf.V <= 64:
        out.append("c planted " + " ".join(str(int(b)) for b in cnf.sigma) + "\n")
    out.append(f"p cnf {cnf.V} {cnf.C}\n")
    head = "".join(out).encode()
    if cnf.C == 0:
        return head
    lens = np.diff(cnf.clause_ptr)
    # interleave literals with a 0 terminator after each clause, vectorised
    term_pos = cnf.clause_ptr[1:] + np.arange(cnf.C)
    total = cnf.nnz + cnf.C
    vals = np.zeros(total, dtype=np.int64)
    is_lit = np.ones(total, dtype=bool)
    is_lit[term_pos] = False
    vals[is_lit] = cnf.lits
    toks = vals.astype(str)
    sep = np.full(total, " ", dtype=object)
    sep[term_pos] = "\n"
    body = "".join((toks.astype(object) + sep).tolist())
    del lens
    return head + body.encode()


def enumeration_theta(V: int) -> np.ndarray:
    """theta (V x 2^V, fp32) with theta[v, n] = +1 if bit v of n is set else -1.

    Every row has mean exactly 0, so Eq. 5's guard is active and the
    binarised batch is exactly the set of all 2^V assignments."""
    n = np.arange(1 << V, dtype=np.int64)
    bits = (n[None, :] >> np.arange(V, dtype=np.int64)[:, None]) & 1
    return np.where(bits == 1, 1.0, -1.0).astype(np.float32)


def random_state(V: int, N: int, seed: int, scale: float = 1.0):
    """Random (theta, m, v) fp32 arrays for state-handoff tests."""
    rng = np.random.default_rng([0x5747E, int(seed), V, N])
    theta = (rng.standard_normal((V, N)) * scale).astype(np.float32)
    m = (rng.standard_normal((V, N)) * 0.05).astype(np.float32)
    v = (rng.random((V, N)) * 0.01).astype(np.float32)
    return theta, m, v


# BASELINE.json "configs", as concrete generator calls.
CONFIGS = {
    "c1": dict(kind="planted", V=20, C=85, k=3, N=64, steps=100, seed=1),
    "c2": dict(kind="planted", V=10_000, C=42_000, k=3, N=4096, steps=360, seed=1),
    "c3": dict(kind="planted", V=1_000_000, C=4_200_000, k=3, N=1024, steps=360, seed=1),
    "c4": dict(kind="industrial", V=500_000, C=2_000_000, N=2048, steps=360, seed=1),
    "c5": dict(kind="planted", V=100_000, C=425_000, k=3, N=65536, steps=3600, seed=1),
    # SURVEY f4 (dense tensor-core tiles) experiment: a small clause-DENSE
    # instance (long clauses over few variables: P is 15/512 = 2.9 % dense) and
    # a sparse one of the same size (3/512 = 0.6 %); not BASELINE configs
    "f4d": dict(kind="planted", V=256, C=4096, k=15, N=8192, steps=360, seed=1),
    "f4s": dict(kind="planted", V=256, C=1075, k=3, N=8192, steps=360, seed=1),
    # c2's shape with 2-hidden planting (not a BASELINE config)
    "c2h": dict(kind="planted", V=10_000, C=42_000, k=3, N=4096, steps=360, seed=1, hidden=2),
}


def make_config(name: str, seed: int | None = None) -> tuple[Cnf, dict]:
    cfg = dict(CONFIGS[name])
    if seed is not None:
        cfg["seed"] = seed
    if cfg["kind"] == "planted":
        cnf = planted_ksat(cfg["V"], cfg["C"], cfg["k"], cfg["seed"], cfg.get("hidden", 1))
    else:
        cnf = industrial_cnf(cfg["V"], cfg["C"], cfg["seed"])
    return cnf, cfg
