"""Native instance generators, DIMACS writer and model checker (host-only
C-ABI, SURVEY §2.8 items 1, 2, 4 and §8(d) "Generators").
Pinned against their definitions: planting (sigma satisfies every clause;
2-hidden: its complement too; per-literal agreement with sigma 4/7 for k = 3,
1/2 for 2-hidden), k distinct variables per clause, the clause-length mix and
the rank^-alpha degree law of the industrial shape, determinism per seed, the
DIMACS writer against the parser and the Python writer, and verify_model
against a direct evaluation."""
import numpy as np
import pytest

from tsat_synth import Cnf, planted_ksat, to_dimacs


def _P():
    from paper_2511_07737_b200 import build
    build.build()
    import paper_2511_07737_b200 as P
    return P


def _direct_unsat(V, ptr, lits, m):
    var = np.abs(lits) - 1
    val = np.where(lits > 0, m[var], 1 - m[var])
    sat = np.add.reduceat(val, ptr[:-1]) > 0 if len(ptr) > 1 else np.zeros(0, bool)
    sat[np.diff(ptr) == 0] = False
    return int((~sat).sum())


@pytest.mark.parametrize("k,hidden", [(3, 1), (3, 2), (5, 1), (15, 1)])
def test_planted_definition(k, hidden):
    P = _P()
    V, C = 3000, 12000
    ptr, lits, sg = P.gen_planted(V, C, k, 11, hidden)
    assert np.array_equal(ptr, np.arange(C + 1) * k) and lits.size == C * k
    L = lits.reshape(C, k)
    assert (np.abs(L) >= 1).all() and (np.abs(L) <= V).all()
    s = np.sort(np.abs(L), axis=1)
    assert (s[:, 1:] != s[:, :-1]).all()                                   # k distinct variables
    assert P.verify_model(V, ptr, lits, sg) == 0                           # sigma is a model
    agree = np.where(L > 0, sg[np.abs(L) - 1] == 1, sg[np.abs(L) - 1] == 0).mean()
    if hidden == 1:
        expect = 2 ** (k - 1) / (2 ** k - 1)                               # 4/7 for k = 3
        assert abs(agree - expect) < 0.01
    else:
        assert P.verify_model(V, ptr, lits, 1 - sg) == 0                   # the complement too
        assert abs(agree - 0.5) < 0.01
    assert 0.45 < sg.mean() < 0.55
    p2, l2, s2 = P.gen_planted(V, C, k, 11, hidden)
    assert np.array_equal(l2, lits) and np.array_equal(s2, sg)            # deterministic
    _, l3, _ = P.gen_planted(V, C, k, 12, hidden)
    assert not np.array_equal(l3, lits)


def test_industrial_shape():
    P = _P()
    V, C = 20000, 80000
    probs = {2: .40, 3: .30, 4: .12, 5: .08, 6: .06, 7: .04}
    ptr, lits, sg = P.gen_industrial(V, C, 5, 0.82, probs)
    lens = np.diff(ptr)
    for k, p in probs.items():
        assert abs((lens == k).mean() - p) < 0.01
    assert P.verify_model(V, ptr, lits, sg) == 0
    for c in range(0, C, 997):                                               # distinct variables
        v = np.abs(lits[ptr[c]:ptr[c + 1]])
        assert len(set(v.tolist())) == len(v)
    deg = np.sort(np.bincount(np.abs(lits) - 1, minlength=V))[::-1].astype(float)
    r = np.arange(1, V + 1)
    sel = (r >= 10) & (r <= 1000)                                            # rank^-alpha over the head
    slope = np.polyfit(np.log(r[sel]), np.log(deg[sel]), 1)[0]
    assert abs(slope + 0.82) < 0.1


def test_dimacs_writer_roundtrip_and_verify():
    P = _P()
    cnf = planted_ksat(40, 170, 3, 2)
    ours = P.write_dimacs(cnf.V, cnf.clause_ptr, cnf.lits, cnf.sigma)
    assert ours == to_dimacs(cnf)                                            # same text as the Python writer
    info = P.parse_dimacs(ours)
    assert (info.V, info.C, info.nnz, info.K) == (cnf.V, cnf.C, cnf.nnz, cnf.K)
    ptr, lits, _ = P.gen_planted(500, 2100, 3, 3)
    big = Cnf(500, ptr, lits)
    txt = P.write_dimacs(big.V, big.clause_ptr, big.lits)
    assert P.parse_dimacs(txt).C == 2100 and not txt.startswith(b"c planted")
    rng = np.random.default_rng(0)
    for _ in range(20):
        m = rng.integers(0, 2, cnf.V).astype(np.uint8)
        assert P.verify_model(cnf.V, cnf.clause_ptr, cnf.lits, m) == _direct_unsat(cnf.V, cnf.clause_ptr, cnf.lits, m)
    e = Cnf.from_clauses(3, [[1, 2], [], [-3]])
    assert P.verify_model(3, e.clause_ptr, e.lits, np.array([1, 0, 0], np.uint8)) == 1   # the empty clause


def test_generator_argument_errors():
    P = _P()
    with pytest.raises(P.TsatError):
        P.gen_planted(10, 5, 11, 1)                     # k > V
    with pytest.raises(P.TsatError):
        P.gen_planted(10, 5, 1, 1, hidden=2)            # 2-hidden needs k >= 2
    with pytest.raises(P.TsatError):
        P.verify_model(3, np.array([0, 1]), np.array([4], np.int32), np.zeros(3, np.uint8))   # |lit| > V


def test_literal_split_relabelling():
    """tsat_synth.literal_split (the 2V-literal-row form of PAPER.md l.191):
    every literal becomes a positive reference to its own literal row; an
    assignment a of the original maps to (a, 1 - a) with identical clause
    truth values, and the planted model maps to a model."""
    from tsat_synth import literal_split
    cnf = planted_ksat(30, 120, 3, 4)
    d = literal_split(cnf)
    assert d.V == 60 and (d.lits > 0).all() and np.array_equal(d.clause_ptr, cnf.clause_ptr)
    rng = np.random.default_rng(1)
    for _ in range(10):
        a = rng.integers(0, 2, cnf.V).astype(np.uint8)
        b = np.concatenate([a, 1 - a])
        assert _direct_unsat(cnf.V, cnf.clause_ptr, cnf.lits, a) == _direct_unsat(d.V, d.clause_ptr, d.lits, b)
    assert _direct_unsat(d.V, d.clause_ptr, d.lits, d.sigma) == 0
