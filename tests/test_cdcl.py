"""CPU CDCL hand-off consumer (§4.2 l.277-287):
tsat_cdcl_solve / tsat_cdcl_portfolio are host-only entry points of
libturbosat.  Pinned against brute-force enumeration (SAT / UNSAT verdicts),
model verification, and the semantics of assumed (seeded) literals."""
import itertools

import numpy as np
import pytest

from tsat_synth import Cnf, fig1_cnf, planted_ksat


def _lib():
    from paper_2511_07737_b200 import build
    build.build()
    import paper_2511_07737_b200 as P
    return P


def _models(cnf):
    """All models by enumeration (V <= 14)."""
    cls = cnf.clauses()
    out = []
    for bits in itertools.product((0, 1), repeat=cnf.V):
        if all(any((bits[abs(x) - 1] == 1) == (x > 0) for x in c) for c in cls):
            out.append(bits)
    return out


def _is_model(cnf, m):
    return all(any((m[abs(x) - 1] == 1) == (x > 0) for x in c) for c in cnf.clauses())


def _random_cnf(V, C, k, seed):
    rng = np.random.default_rng(seed)
    cl = []
    for _ in range(C):
        vs = rng.choice(V, size=k, replace=False) + 1
        cl.append([int(v) * (1 if rng.random() < 0.5 else -1) for v in vs])
    return Cnf.from_clauses(V, cl)


@pytest.mark.parametrize("seed", range(12))
def test_verdicts_match_brute_force(seed):
    P = _lib()
    V = 10 + seed % 4
    cnf = _random_cnf(V, int(V * (3.5 + 0.25 * (seed % 8))), 3, seed)     # both SAT and UNSAT instances
    models = _models(cnf)
    for s in (0, seed + 1):
        res, m = P.cdcl_solve(cnf, seed=s)
        if models:
            assert res.status == 10 and _is_model(cnf, m)
        else:
            assert res.status == 20 and m is None


def test_fig1_and_trivial_cases():
    P = _lib()
    res, m = P.cdcl_solve(fig1_cnf())
    assert res.status == 10 and tuple(m) in {(1, 0, 0, 1), (1, 1, 0, 1)}      # TFFT, TTFT (R16)
    assert P.cdcl_solve(Cnf.from_clauses(1, [[1], [-1]]))[0].status == 20
    assert P.cdcl_solve(Cnf.from_clauses(3, [[1, 2], []]))[0].status == 20     # empty clause
    assert P.cdcl_solve(Cnf.from_clauses(3, []))[0].status == 10
    assert P.cdcl_solve(Cnf.from_clauses(2, [[1, -1], [2]]))[0].status == 10   # tautology kept harmless


def test_assumptions_seed_the_search():
    """Assumed literals are fixed (l.291: assigning V* variables prunes the
    space by 2^V*): consistent seeds give a model that extends them; seeds
    excluding every model give status 21, never a wrong model."""
    P = _lib()
    cnf = _random_cnf(12, 40, 3, 5)
    models = _models(cnf)
    assert models
    m0 = models[0]
    seed_lits = [(v + 1) if m0[v] else -(v + 1) for v in range(4)]
    res, m = P.cdcl_solve(cnf, seed_lits)
    assert res.status == 10 and _is_model(cnf, m)
    assert all((m[abs(x) - 1] == 1) == (x > 0) for x in seed_lits)
    for trial in range(20):                                  # random 5-literal seeds vs enumeration
        rng = np.random.default_rng(trial)
        vs = rng.choice(12, 5, replace=False)
        lits = [int(v + 1) * (1 if rng.random() < .5 else -1) for v in vs]
        ext = [b for b in models if all((b[abs(x) - 1] == 1) == (x > 0) for x in lits)]
        res, m = P.cdcl_solve(cnf, lits)
        assert res.status == (10 if ext else 21)
        if ext:
            assert tuple(m) in set(ext)


def test_portfolio_seeded_and_failing_seeds():
    P = _lib()
    cnf = planted_ksat(150, 600, 3, 7)
    sig = cnf.sigma
    good = [[(v + 1) if sig[v] else -(v + 1) for v in range(20)]]
    res, m = P.cdcl_portfolio(cnf, np.array(good, np.int32), threads=2, unseeded=False, time_limit_s=30)
    assert res.status == 10 and res.winner == 0 and _is_model(cnf, m)
    # seeds that contradict a unit clause fail; the unseeded instance still solves
    cnf2 = Cnf.from_clauses(cnf.V, cnf.clauses() + [[1 if sig[0] else -1]])
    bad = np.array([[-1 if sig[0] else 1] + [0] * 19] * 3, np.int32)
    res, m = P.cdcl_portfolio(cnf2, bad, threads=1, unseeded=True, time_limit_s=30)
    assert res.status == 10 and _is_model(cnf2, m)
    res, m = P.cdcl_portfolio(cnf2, bad, threads=2, unseeded=False, time_limit_s=30)
    assert res.status == 0 and res.failed_seeds == 3 and m is None


def test_argument_errors():
    P = _lib()
    cnf = fig1_cnf()
    with pytest.raises(P.TsatError):
        P.cdcl_solve(cnf, [7])                              # |lit| > V
    bad = Cnf(4, np.array([0, 2, 1], np.int64), np.array([1, 2], np.int32))
    with pytest.raises(P.TsatError):
        P.cdcl_solve(bad)                                   # non-monotone offsets
    with pytest.raises(P.TsatError):
        P.cdcl_portfolio(cnf, np.zeros((1, 2), np.int32), threads=0)
