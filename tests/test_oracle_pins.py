"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test names the passage it pins (PAPER.md line / section / equation) and
uses a check that is independent of the oracle's own code: paper values,
brute-force enumeration, high-precision (mpmath) evaluation, torch autograd of
the dense formulation, torch.optim.AdamW, closed forms and invariants.
"""
import itertools
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from tsat_synth import Cnf, enumeration_theta, fig1_cnf, industrial_cnf, planted_ksat

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, *vals = line.split()
        out[k] = vals
    return out


def _direct_eval(cnf, assignment):
    """Clause-by-clause satisfied-literal counts (independent of the oracle)."""
    return [sum(1 for x in cl if (assignment[abs(x) - 1] == 1) == (x > 0)) for cl in cnf.clauses()]


# ------------------------------------------------------------ Philox / init
def test_philox_known_answers():
    """Random123 Philox4x32-10 KAT vectors (golden/philox_kat.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLD, "philox_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        vals = [int(x, 16) for x in r]
        out = O.philox(vals[0:4], vals[4:6])
        assert [int(x) for x in out] == vals[6:10]


def test_init_statistics_and_shard_invariance():
    """PAPER.md §4.1 l.250-252: theta0 ~ N(0,1) gives ~half True literals."""
    from scipy import stats
    V, N = 1000, 64
    th, m, v = O.init_theta(V, N, seed=7)
    assert not m.any() and not v.any()
    frac = (th > 0).mean()
    assert 0.45 <= frac <= 0.55
    assert abs(th.mean()) < 4 / math.sqrt(V * N)
    assert abs(th.std() - 1) < 0.02
    assert stats.kstest(th.ravel().astype(np.float64), "norm").pvalue > 1e-3
    th2, _, _ = O.init_theta(V, N, seed=7)
    assert np.array_equal(th, th2)                           # determinism
    a, _, _ = O.init_theta(V, N, seed=7, n0=24, Nl=20)       # a shard = a slice
    assert np.array_equal(a, th[:, 24:44])
    b, _, _ = O.init_theta(V, N, seed=8)
    assert not np.array_equal(th, b)


# ------------------------------------------------------------ Fig. 1/2
def test_fig2_result_matrix_entries():
    """PAPER.md §3.1.3 l.161-167: R[3,2] = 0 and R[3,3] = 2; l.148 clause 2."""
    gd = _golden("fig2.txt")
    cnf = fig1_cnf()
    assert sorted(cnf.clauses()[1]) == [int(x) for x in gd["clause2"]]
    cols = ["1001", "1110", "0001"]
    b = np.array([[int(c[v]) for c in cols] for v in range(4)], np.uint8)
    R = O.clause_eval(cnf, b)
    assert R[2, 1] == int(gd["R_3_2"][0])
    assert R[2, 2] == int(gd["R_3_3"][0])
    assert R[1, 1] == int(gd["R_2_2"][0])
    assert R[:, 1].tolist() == [int(x) for x in gd["Rcol2"]]
    # column 1 is a model: every clause has a true literal (Fig. 1 caption l.50)
    assert R[:, 0].min() >= 1
    assert R[:, 0].tolist() == _direct_eval(cnf, [1, 0, 0, 1])


def test_fig1_models_by_enumeration():
    """§3.1.4 l.169-177: SAT iff the column minimum is nonzero.  Enumerate all
    16 assignments of the Fig. 1 reconstruction."""
    gd = _golden("fig2.txt")
    cnf = fig1_cnf()
    th = enumeration_theta(4)
    o = O.Oracle(cnf, 16, seed=0, init=False)
    o.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
    s = o.step()
    models = {"".join(str(int(s.bits[v, n])) for v in range(4)) for n in range(16) if s.unsat[n] == 0}
    assert models == set(gd["models"])


# ------------------------------------------------------------ brute force
@pytest.mark.parametrize("V,C,seed", [(8, 30, 1), (10, 45, 2), (12, 60, 3)])
def test_clause_eval_brute_force_small(V, C, seed):
    """Every assignment: oracle R equals direct clause-by-clause evaluation."""
    cnf = planted_ksat(V, C, 3, seed)
    th = enumeration_theta(V)
    o = O.Oracle(cnf, 1 << V, seed=0, init=False)
    o.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
    s = o.step()
    for n in range(0, 1 << V, 37):
        a = [(n >> v) & 1 for v in range(V)]
        assert s.bits[:, n].tolist() == a
        assert s.R[:, n].tolist() == _direct_eval(cnf, a)
        assert s.unsat[n] == sum(1 for r in _direct_eval(cnf, a) if r == 0)


@pytest.mark.parametrize("V,C,k,seed", [(12, 20, 9, 1), (16, 12, 12, 2), (15, 4, 15, 3)])
def test_clause_eval_brute_force_long_clauses(V, C, k, seed):
    """SURVEY f3 (K > 7, R in 0..15): every assignment's R and unsat count
    equal direct clause-by-clause evaluation."""
    cnf = planted_ksat(V, C, k, seed)
    th = enumeration_theta(V)
    o = O.Oracle(cnf, 1 << V, seed=0, init=False)
    o.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
    s = o.step()
    assert s.h.shape[1] == k + 1
    for n in range(0, 1 << V, 97):
        a = [(n >> v) & 1 for v in range(V)]
        assert s.R[:, n].tolist() == _direct_eval(cnf, a)
        assert s.unsat[n] == sum(1 for r in _direct_eval(cnf, a) if r == 0)


def test_enumeration_batch_v20():
    """north_star: brute-force enumeration of all 2^20 assignments of a planted
    20-variable instance (config c1 shape).  Unsat counts from the oracle equal
    a vectorised direct evaluation; min unsat = 0 (the planted model)."""
    cnf = planted_ksat(20, 85, 3, 1)
    V = 20
    n = np.arange(1 << V, dtype=np.int64)
    lits = np.array(cnf.clauses())
    var = np.abs(lits) - 1
    vals = ((n[None, None, :] >> var[:, :, None]) & 1) == (lits[:, :, None] > 0)
    unsat_direct = (~vals.any(axis=1)).sum(axis=0)
    th = enumeration_theta(V)
    o = O.Oracle(cnf, 1 << V, seed=0, init=False)
    o.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
    s = o.step()
    assert np.array_equal(s.unsat, unsat_direct)
    assert s.unsat.min() == 0
    sigma_idx = int(sum(int(b) << v for v, b in enumerate(cnf.sigma)))
    assert s.unsat[sigma_idx] == 0
    assert s.best_unsat == 0


@pytest.mark.parametrize("maker", [lambda: planted_ksat(40, 170, 3, 5), lambda: industrial_cnf(200, 600, 3)])
def test_histogram_invariants(maker):
    """sum_r h_r = C; sum_r r h_r = sum over variables of true-literal
    occurrences (double counting); R <= clause length; zero unsat => model."""
    cnf = maker()
    o = O.Oracle(cnf, 96, seed=3)
    for _ in range(3):
        s = o.step()
        assert (s.h.sum(axis=1) == cnf.C).all()
        lens = np.diff(cnf.clause_ptr)
        assert (s.R <= lens[:, None]).all()
        var = np.abs(cnf.lits) - 1
        pos = cnf.lits > 0
        occp = np.bincount(var[pos], minlength=cnf.V)
        occn = np.bincount(var[~pos], minlength=cnf.V)
        truth = (s.bits * occp[:, None] + (1 - s.bits) * occn[:, None]).sum(axis=0)
        assert np.array_equal((s.h * np.arange(cnf.K + 1)).sum(axis=1), truth)
        for n in np.nonzero(s.unsat == 0)[0]:
            assert min(_direct_eval(cnf, s.bits[:, n].tolist())) >= 1


# ------------------------------------------------------------ SmoothMin
def _mp_smoothmin(col, tau):
    import mpmath as mp
    mp.mp.dps = 40
    w = [mp.e ** (-mp.mpf(tau) * r) for r in col]
    return sum(mp.mpf(r) * x for r, x in zip(col, w)) / sum(w)


@pytest.mark.parametrize("tau", [0.5, 1.0, 5.0])
def test_smoothmin_high_precision_fig1(tau):
    """Eq. 4 on Fig. 1 column 2 (R = [2,1,0,0,2]) against a
    40-digit mpmath evaluation of the formula as printed."""
    col = [2, 1, 0, 0, 2]
    h = np.array([[2, 1, 2, 0]], np.int32)  # counts of R = 0,1,2,3 (K=3)
    S, g, rmin = O.smoothmin(h, tau)
    ref = float(_mp_smoothmin(col, tau))
    assert abs(S[0] - ref) <= 4e-16 * max(1.0, abs(ref))
    assert abs(O.smoothmin_direct(col, tau) - ref) <= 4e-16 * max(1.0, abs(ref))


def test_smoothmin_derivative_high_precision():
    """dS/dR_c (the table g) against mpmath numerical differentiation of Eq. 4;
    translation equivariance sum_c dS/dR_c = 1."""
    import mpmath as mp
    mp.mp.dps = 40
    col = [2, 1, 0, 0, 2]
    h = np.array([[2, 1, 2, 0]], np.int32)
    for tau in (0.5, 1.0, 5.0):
        _, g, _ = O.smoothmin(h, tau)

        def S(*R):
            w = [mp.e ** (-mp.mpf(tau) * r) for r in R]
            return sum(r * x for r, x in zip(R, w)) / sum(w)

        grads = []
        for c in range(5):
            d = [0] * 5
            d[c] = 1
            grads.append(float(mp.diff(S, [mp.mpf(x) for x in col], tuple(d))))
        ours = [g[0, r] for r in col]
        np.testing.assert_allclose(ours, grads, rtol=1e-14, atol=1e-16)
        assert abs(sum(ours) - 1.0) < 1e-14
    # survey's derived values at tau = 1
    _, g, _ = O.smoothmin(h, 1.0)
    np.testing.assert_allclose([g[0, r] for r in col],
                               [-0.0336169346751, 0.0480445481544, 0.509594660598, 0.509594660598, -0.0336169346751],
                               rtol=1e-10)


def test_smoothmin_closed_forms_and_grouping():
    """Constant column -> its value; S in [min, max]; tau -> inf gives min;
    grouped (histogram) form equals the direct C-term sum to rounding."""
    rng = np.random.default_rng(0)
    for k in range(4):
        h = np.zeros((1, 4), np.int32)
        h[0, k] = 17
        S, g, _ = O.smoothmin(h, 1.0)
        assert S[0] == k
        assert abs(g[0, k] * 17 - 1.0) < 1e-15      # uniform weights 1/17
    for _ in range(50):
        col = rng.integers(0, 4, size=rng.integers(1, 200)).astype(np.int32)
        h = np.bincount(col, minlength=4).astype(np.int32)[None, :]
        for tau in (0.3, 1.0, 7.0):
            S, _, _ = O.smoothmin(h, tau)
            assert col.min() - 1e-12 <= S[0] <= col.max() + 1e-12
            assert abs(S[0] - O.smoothmin_direct(col, tau)) <= 1e-13 * max(1, S[0])
    S, _, _ = O.smoothmin(np.array([[1, 0, 0, 0, 0, 1]], np.int32), 1000.0)
    assert S[0] < 1e-6  # column [0, 5]


def test_loss_all_equal():
    """Eq. 3: all R entries equal k gives L = -N k."""
    cnf = Cnf.from_clauses(3, [[1, 2, 3]] * 5)
    th = np.ones((3, 8), np.float32)                   # mu = 1 > 0: all True -> R = 3
    o = O.Oracle(cnf, 8, 0, init=False)
    o.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
    s = o.step()
    assert s.loss == -8 * 3.0
    assert (s.unsat == 0).all()


# ------------------------------------------------------------ gradient chain
def _torch_dense_grad(cnf, theta, tau, normalize=True, eps=1e-8):
    """Dense fp64 torch autograd of the paper's graph (Fig. 3): Eq. 5 normalise,
    Eq. 2 binarise with STE, R = P A (Eq. 1, 2V literal rows), Eq. 4, Eq. 3."""
    import torch
    V, N = theta.shape
    Pp = torch.zeros(cnf.C, V, dtype=torch.float64)
    Pn = torch.zeros(cnf.C, V, dtype=torch.float64)
    for c, cl in enumerate(cnf.clauses()):
        for x in cl:
            (Pp if x > 0 else Pn)[c, abs(x) - 1] = 1.0
    th = torch.tensor(theta.astype(np.float64), requires_grad=True)
    if normalize == 3:                       # R28: mean magnitude (variant f2)
        d = torch.clamp(th.abs().mean(dim=1, keepdim=True), min=eps)
        x = th / d
    elif normalize:
        mu = th.mean(dim=1, keepdim=True)
        mag = torch.clamp(mu.abs(), min=eps)
        d = torch.where(mu >= 0, mag, -mag)
        x = th / d
    else:
        x = th
    B = (x > 0).to(torch.float64)
    a = x + (B - x).detach()                 # STE
    R = Pp @ a + Pn @ (1 - a)                # R = P A with A_neg = 1 - A_pos
    w = torch.exp(-tau * (R - R.detach().min(dim=0).values))
    S = (R * w).sum(0) / w.sum(0)
    L = -S.sum()
    L.backward()
    return th.grad.numpy(), float(L)


def _G_from_g64(cnf, R, g):
    """G_vn = sum_{c contains -v} g_n[R_cn] - sum_{c contains +v} g_n[R_cn] (numpy)."""
    G = np.zeros((cnf.V, R.shape[1]))
    cols = np.arange(R.shape[1])
    for c, cl in enumerate(cnf.clauses()):
        vals = g[cols, R[c]]
        for x in cl:
            G[abs(x) - 1] += vals if x < 0 else -vals
    return G


@pytest.mark.parametrize("seed,tau,normalize", [(1, 1.0, 1), (2, 0.5, 1), (3, 5.0, 1), (4, 1.0, 0), (5, 2.0, 1),
                                                (6, 1.0, 3), (7, 2.0, 3), (8, 1.0, 1), (9, 0.5, 1)])
def test_gradient_matches_torch_autograd(seed, tau, normalize):
    """STE backward + Eq. 5 Jacobian
    against torch autograd of the dense formulation, fp64.  Seeds 8 and 9 use
    long clauses (K = 12 and a 2..15 mix: SURVEY f3)."""
    rng = np.random.default_rng(seed)
    V, C, N = 10, 40, 24
    if seed == 8:
        V, C = 16, 30
        cnf = planted_ksat(V, C, 12, seed)
    elif seed == 9:
        V = 24
        cl = planted_ksat(V, 8, 15, seed).clauses() + planted_ksat(V, 10, 9, seed).clauses()
        cl += planted_ksat(V, 30, 3, seed).clauses() + planted_ksat(V, 10, 2, seed).clauses()
        from tsat_synth import Cnf
        cnf = Cnf.from_clauses(V, cl)
    else:
        cnf = planted_ksat(V, C, 3, seed) if seed % 2 else industrial_cnf(V, C, seed)
    theta = (np.round(rng.standard_normal((V, N)) * 2 ** 16) / 2 ** 16).astype(np.float32)
    theta[:, 0] += 0.2                           # keep |mu| away from the guard
    cfg = O.Config(tau=tau, normalize=normalize)
    o = O.Oracle(cnf, N, 0, cfg=cfg, init=False)
    assert o.cnf is cnf
    o.set_state(theta, np.zeros_like(theta), np.zeros_like(theta), 0)
    s = o.step()
    ref, Lref = _torch_dense_grad(cnf, theta, tau, normalize)
    sgn = np.sign(theta).astype(np.float64) if normalize == 3 else 1.0
    ours = s.G * s.extra["rho"][:, None] - sgn * s.extra["cv"][:, None]
    # element by element (the fp32 g table R26 and fp32 G R27 round each P^T
    # term): 1e-5 relative, floor 2^-20 x the magnitude of the summed terms
    # (tests/test_oracle_pins2.py states the criterion)
    from test_oracle_pins2 import _check_elementwise, _pt_abs
    terms = _pt_abs(o.cnf, s.R, s.g) * np.abs(s.extra["rho"][:, None]) + np.abs(s.extra["cv"][:, None])
    _check_elementwise(ours, ref, terms, "G rho - c")
    _check_elementwise(s.grad, ref, terms, "fp32 grad")
    # G itself is the P^T fold (numpy, fp64 table) up to the fp32 rounding of g
    G64 = _G_from_g64(o.cnf, s.R, s.g)
    assert np.abs(s.G - G64).max() <= 2.4e-7 * np.abs(G64).max()
    G32 = _G_from_g64(o.cnf, s.R, s.g32.astype(np.float64))
    assert np.abs(s.G - G32).max() <= 4 * 2.0 ** -24 * np.abs(G32).max()
    assert abs(s.loss - Lref) <= 1e-12 * abs(Lref)
    _assert_fp32_fma(s.grad, s.G, s.extra["rho"], s.extra["cv"], theta if normalize == 3 else None)


def _assert_fp32_fma(grad, G, rho, cv, theta=None):
    """R27b: grad = fmaf(G, (float)rho, -(float)c), i.e. the exact value
    G rho_f - c_f correctly rounded to fp32 (|err| <= 1/2 ulp, exact rationals)."""
    from fractions import Fraction
    rf = rho.astype(np.float32)
    cf = cv.astype(np.float32)
    for v in range(G.shape[0]):
        for j in range(G.shape[1]):
            g = np.float32(grad[v, j])
            c = Fraction(float(cf[v]))
            if theta is not None:                 # R28: the Jacobian term carries sign(theta)
                c = c * int(np.sign(theta[v, j]))
            exact = Fraction(float(np.float32(G[v, j]))) * Fraction(float(rf[v])) - c
            half_ulp = Fraction(float(np.spacing(np.abs(g)))) / 2
            assert abs(Fraction(float(g)) - exact) <= half_ulp, (v, j)


@pytest.mark.parametrize("normalize", [1, 3])
def test_euler_invariant(normalize):
    """Eq. 5 is scale invariant per row (also with the mean-magnitude
    denominator, R28), so sum_n theta_vn dL/dtheta_vn = 0.
    (theta on a 2^-20 grid so the fixed-point row mean, R10, is exact.)"""
    cnf = planted_ksat(50, 210, 3, 9)
    rng = np.random.default_rng(4)
    th = (np.round(rng.standard_normal((50, 128)) * 2 ** 20) / 2 ** 20).astype(np.float32)
    o = O.Oracle(cnf, 128, seed=0, init=False, cfg=O.Config(normalize=normalize))
    o.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
    s = o.step()
    th = th.astype(np.float64)
    sgn = np.sign(th) if normalize == 3 else 1.0
    ours = s.G * s.extra["rho"][:, None] - sgn * s.extra["cv"][:, None]
    lhs = (th * ours).sum(axis=1)
    scale = np.abs(th * ours).sum(axis=1) + 1e-300
    act = s.extra["guard"] == 0
    assert act.all()
    # sum theta grad = rho (J_exact - J): only J's fixed-point rounding remains
    # (R13: fp32 products, 2^-24 relative, and the 2^-(s+1) integer rounding)
    jerr = np.abs(s.G * th).sum(axis=1) * 2.0 ** -24 + 128 * 2.0 ** (-s.extra["s"].astype(np.float64) - 1)
    assert (np.abs(lhs) <= np.abs(s.extra["rho"]) * jerr + 1e-12 * scale).all()
    assert (np.abs(lhs) <= 1e-6 * scale).all()


def test_repeated_literal_is_one_matrix_entry():
    """§3.1.1 l.146-147: P holds only 0/1, so (x4 v x4 v ~x5) evaluates exactly
    like (x4 v ~x5)."""
    a = Cnf.from_clauses(5, [[4, 4, -5], [1, 2, 3]])
    b = Cnf.from_clauses(5, [[4, -5], [1, 2, 3]])
    th = enumeration_theta(5)
    outs = []
    for cnf in (a, b):
        o = O.Oracle(cnf, 32, 0, init=False)
        o.set_state(th, np.zeros_like(th), np.zeros_like(th), 0)
        outs.append(o.step())
    np.testing.assert_array_equal(outs[0].R, outs[1].R)
    assert outs[0].R[0].max() == 2 and o.K == 3


def test_tautology_and_unit_special_cases():
    """A tautology (x v ~x) contributes 0 to G; a unit clause (x1) pushes x1
    toward True; N = 1 gives a zero gradient (x = theta/mean = 1)."""
    cnf = Cnf.from_clauses(2, [[1, -1], [2]])
    theta = np.array([[0.5, -0.25, 1.0, -2.0], [0.3, -0.7, 0.2, 0.1]], np.float32)
    o = O.Oracle(cnf, 4, 0, cfg=O.Config(normalize=0), init=False)
    o.set_state(theta, np.zeros_like(theta), np.zeros_like(theta), 0)
    s = o.step()
    assert (s.G[0] == 0).all()
    assert (s.G[1] < 0).all()          # dL/dx2 < 0: increasing x2 lowers the loss
    o1 = O.Oracle(cnf, 1, 0, init=False)
    t1 = np.array([[0.7], [-0.4]], np.float32)
    o1.set_state(t1, np.zeros_like(t1), np.zeros_like(t1), 0)
    s1 = o1.step()
    assert (s1.grad == 0).all()
    assert s1.bits[:, 0].tolist() == [1, 1]


def test_jacobian_fixed_point_is_exact_sum():
    """J_v = sum_m G_vm theta_vm: the int64 fixed point (R13: fp32 products,
    each rounded to an integer at scale 2^s_v) equals the exact sum
    (math.fsum) to within sum |G theta| 2^-24 + N 2^-(s_v+1)."""
    cnf = planted_ksat(30, 126, 3, 4)
    o = O.Oracle(cnf, 64, seed=5)
    th = o.theta.astype(np.float64).copy()
    s = o.step()
    for v in range(cnf.V):
        exact = math.fsum((s.G[v] * th[v]).tolist())
        sv = int(s.extra["s"][v])
        assert -126 <= sv <= 127
        bound = np.abs(s.G[v] * th[v]).sum() * 2.0 ** -24 + 64 * 2.0 ** (-sv - 1)
        assert abs(s.J[v] - exact) <= bound + 1e-300
        # s_v is the largest scale that keeps N occ gmax thmax 2^s_v <= 2^61
        assert np.abs(s.G[v] * th[v]).max() * 2.0 ** sv <= 2.0 ** 61


def test_moment_reset_is_a_fresh_optimizer():
    """Variant f2: with reset_moments_on_restart the iteration
    at an LR restart equals the first iteration of a freshly created AdamW
    (m = v = 0, step 1, lr0) from the same theta; without it, it does not."""
    cnf = planted_ksat(40, 170, 3, 2)
    N = 64
    cfg = O.Config(reset_moments_on_restart=1, restart_every=5, decay_every=2)
    o = O.Oracle(cnf, N, seed=11, cfg=cfg)
    for _ in range(5):
        o.step()
    assert o.t == 5 and np.abs(o.m).max() > 0
    th5 = o.theta.copy()
    fresh = O.Oracle(cnf, N, seed=11, cfg=cfg, init=False)
    fresh.set_state(th5, np.zeros_like(th5), np.zeros_like(th5), 0)
    o.step()
    fresh.step()
    np.testing.assert_array_equal(o.theta, fresh.theta)
    np.testing.assert_array_equal(o.m, fresh.m)
    np.testing.assert_array_equal(o.v, fresh.v)
    plain = O.Oracle(cnf, N, seed=11, cfg=O.Config(restart_every=5, decay_every=2))
    for _ in range(6):
        plain.step()
    assert not np.array_equal(plain.theta, o.theta)
    # before the first restart the two runs coincide
    a = O.Oracle(cnf, N, seed=11, cfg=cfg)
    b = O.Oracle(cnf, N, seed=11, cfg=O.Config(restart_every=5, decay_every=2))
    for _ in range(5):
        a.step(); b.step()
    np.testing.assert_array_equal(a.theta, b.theta)


# ------------------------------------------------------------ AdamW / LR
def test_lr_schedule():
    """PAPER.md §4.1 l.255-259 (0-based iterations, R9)."""
    cfg = O.Config()
    assert O.lr_at(0, cfg) == 0.1
    assert O.lr_at(29, cfg) == 0.1
    assert math.isclose(O.lr_at(30, cfg), 1e-2, rel_tol=1e-15)
    assert math.isclose(O.lr_at(59, cfg), 1e-2, rel_tol=1e-15)
    assert math.isclose(O.lr_at(60, cfg), 1e-3, rel_tol=1e-15)
    assert math.isclose(O.lr_at(359, cfg), 1e-12, rel_tol=1e-15)
    assert O.lr_at(360, cfg) == 0.1
    assert O.lr_at(720 + 31, cfg) == O.lr_at(31, cfg)
    lo = O.Config(restart_every=480)
    assert O.lr_at(450, lo) == 1e-15                       # the 1e-15 floor binds only past 420


def test_adamw_matches_torch():
    """torch.optim.AdamW (defaults, R6) fed the same gradient sequence across
    an LR decay boundary: identical up to torch's CPU sqrt rounding."""
    import torch
    V, N = 8, 64
    rng = np.random.default_rng(3)
    th0 = rng.standard_normal((V, N)).astype(np.float32)
    p = torch.nn.Parameter(torch.tensor(th0.copy()))
    opt = torch.optim.AdamW([p], lr=0.1)
    th, m, v = th0.copy(), np.zeros_like(th0), np.zeros_like(th0)
    cfg = O.Config()
    L = O.lib()
    for t in range(40):
        g = (rng.standard_normal((V, N)) * 10 ** rng.uniform(-3, 1)).astype(np.float32)
        lr = O.lr_at(t, cfg)
        for gr in opt.param_groups:
            gr["lr"] = lr
        p.grad = torch.tensor(g)
        opt.step()
        L.or_adamw(V, 0, N, O._p(th), O._p(m), O._p(v), O._p(g), t, t + 1, lr, 0.9, 0.999, 1e-8, 1e-2, 0.0, 0)
        st = opt.state[p]
        np.testing.assert_allclose(st["exp_avg"].numpy(), m, rtol=0, atol=0)
        np.testing.assert_allclose(st["exp_avg_sq"].numpy(), v, rtol=0, atol=0)
        # theta: torch's CPU sqrt is not correctly rounded and R6c multiplies by
        # 1/sqrt(bc2) instead of dividing: each step may differ by ~1 ulp of the
        # update (<= 0.3 here), which weight decay carries forward over 40 steps
        np.testing.assert_allclose(p.detach().numpy(), th, rtol=2e-6, atol=2e-6)


def test_adamw_closed_forms():
    """Zero grad with wd = 0 leaves theta unchanged; a constant gradient gives
    steps of magnitude -> lr (Adam's unit-step property)."""
    V, N = 2, 32
    th = np.full((V, N), 0.75, np.float32)
    m = np.zeros_like(th); v = np.zeros_like(th)
    g = np.zeros_like(th)
    L = O.lib()
    for t in range(5):
        L.or_adamw(V, 0, N, O._p(th), O._p(m), O._p(v), O._p(g), t, t + 1, 0.1, 0.9, 0.999, 1e-8, 0.0, 0.0, 0)
    assert (th == 0.75).all()
    g = np.full((V, N), 0.5, np.float32)
    prev = th.copy()
    for t in range(200):
        L.or_adamw(V, 0, N, O._p(th), O._p(m), O._p(v), O._p(g), t, t + 1, 0.01, 0.9, 0.999, 1e-8, 0.0, 0.0, 0)
        step = prev - th
        prev = th.copy()
    assert abs(step.mean() - 0.01) < 1e-4


# ------------------------------------------------------------ selection / export
def test_compute_k_and_export_order():
    """k = 0.01% of V but >= 20 (<= V); smallest |grad|
    first, ties to the lower variable."""
    assert O.compute_k(1_000_000) == 100
    assert O.compute_k(10_000) == 20
    assert O.compute_k(12) == 12
    assert O.compute_k(200_001) == 21
    lits, mags = O.export_partial(np.array([0.5, 0.0, 0.3, 0.9]), np.array([1, 0, 1, 1], np.uint8), 2)
    assert lits.tolist() == [-2, 3]
    lits, _ = O.export_partial(np.array([0.1, 0.1, 0.0]), np.array([1, 1, 1], np.uint8), 3)
    assert lits.tolist() == [3, 1, 2]


def test_select_top_stable():
    """prioritise candidates with more satisfied clauses;
    ties -> lower index."""
    unsat = np.array([3, 1, 2, 1, 0, 2], np.int32)
    idx, u = O.select_top(unsat, 4)
    assert idx.tolist() == [4, 1, 3, 2]
    assert u.tolist() == [0, 1, 1, 2]


# ------------------------------------------------------------ end to end
def test_fig1_end_to_end_solves():
    """The Fig. 1 instance is satisfiable (l.50); N = 8 candidates reach a model
    in {TFFT, TTFT} and the model verifies."""
    o = O.Oracle(fig1_cnf(), 8, seed=1)
    for _ in range(200):
        s = o.step()
        if s.best_unsat == 0:
            break
    assert s.best_unsat == 0
    a = s.bits[:, s.best_idx].tolist()
    assert "".join(map(str, a)) in ("1001", "1101")
    assert min(_direct_eval(fig1_cnf(), a)) >= 1


def test_unsat_core_never_solves():
    """(x1) ^ (~x1): no candidate satisfies both; best fraction stays 0.5."""
    o = O.Oracle(Cnf.from_clauses(1, [[1], [-1]]), 32, seed=2)
    for _ in range(60):
        s = o.step()
        assert s.best_unsat == 1
        assert np.isfinite(o.theta).all()


class ThreadComm:
    """W ranks as threads; collectives through a barrier (ctypes releases the
    GIL, so the shards really run concurrently)."""

    def __init__(self, world):
        import threading
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world

    def rank(self, r):
        comm = self

        class R:
            def _coll(self, x, fn):
                comm.slots[r] = x
                comm.bar.wait()
                out = fn(list(comm.slots))
                comm.bar.wait()
                return out

            def sum_i64(self, a):
                return self._coll(a.copy(), lambda xs: np.sum(np.stack(xs), axis=0, dtype=np.int64))

            def max(self, x):
                return self._coll(x, max)

            def min_key(self, k):
                return self._coll(k, min)

            def gather_f64(self, a):
                return self._coll(a.copy(), np.concatenate)

        return R()


def run_sharded(cnf, N, seed, world, steps, cfg=None):
    import threading
    comm = ThreadComm(world)
    Nl = N // world
    shards = [O.Oracle(cnf, N, seed, cfg=cfg, n0=r * Nl, Nl=Nl) for r in range(world)]
    for r, o in enumerate(shards):
        o.comm = comm.rank(r)
    outs = [[None] * world for _ in range(steps)]

    def work(r):
        for t in range(steps):
            outs[t][r] = shards[r].step()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [x.start() for x in th]
    [x.join() for x in th]
    return shards, outs


def test_per_shard_normalisation_is_independent_shards():
    """Variant f2 normalize = 2: W = 2 shards normalising over their own
    candidates evolve exactly like two independent single-shard runs
    (normalize = 1, N = N/2) on the candidate slices; best and loss are still
    the global ones.  With W = 1 it is the default (normalize = 1)."""
    cnf = planted_ksat(50, 212, 3, 6)
    N, T = 64, 8
    shards, outs = run_sharded(cnf, N, 4, 2, T, cfg=O.Config(normalize=2))
    init = O.Oracle(cnf, N, seed=4)
    for r in range(2):
        sl = slice(32 * r, 32 * (r + 1))
        ind = O.Oracle(cnf, 32, seed=0, init=False)
        ind.set_state(init.theta[:, sl], init.m[:, sl], init.v[:, sl], 0)
        for t in range(T):
            st = ind.step()
            assert np.array_equal(outs[t][r].unsat, st.unsat)
        assert np.array_equal(ind.theta, shards[r].theta)
    for t in range(T):
        u = np.concatenate([o.unsat for o in outs[t]])
        j = int(np.lexsort((np.arange(N), u))[0])
        assert (outs[t][1].best_unsat, outs[t][1].best_idx) == (int(u[j]), j)
    # the global-normalisation run differs
    g_shards, _ = run_sharded(cnf, N, 4, 2, T)
    assert not np.array_equal(g_shards[0].theta, shards[0].theta)
    one = O.Oracle(cnf, N, seed=4, cfg=O.Config(normalize=2))
    ref = O.Oracle(cnf, N, seed=4)
    for _ in range(4):
        one.step(); ref.step()
    assert np.array_equal(one.theta, ref.theta)


@pytest.mark.parametrize("normalize", [1, 3])
def test_trajectory_determinism_and_shard_invariance(normalize):
    """Same (instance, seed) twice gives identical trajectories; 2- and 4-shard
    runs (candidate sharding) equal the 1-shard run bit for bit
    (global Eq. 5 and its mean-magnitude reading R28)."""
    cnf = planted_ksat(60, 255, 3, 2)
    N, T = 64, 12
    cfg = O.Config(normalize=normalize)
    a = O.Oracle(cnf, N, seed=9, cfg=cfg)
    b = O.Oracle(cnf, N, seed=9, cfg=cfg)
    ref = []
    for t in range(T):
        sa, sb = a.step(), b.step()
        assert np.array_equal(a.theta, b.theta) and sa.loss == sb.loss
        ref.append((a.theta.copy(), sa))
    for world in (2, 4):
        shards, outs = run_sharded(cnf, N, 9, world, T, cfg=cfg)
        th = np.concatenate([o.theta for o in shards], axis=1)
        assert np.array_equal(th, a.theta)
        for t in range(T):
            sa = ref[t][1]
            assert np.array_equal(np.concatenate([o.unsat for o in outs[t]]), sa.unsat)
            assert outs[t][0].loss == sa.loss
            assert (outs[t][0].best_unsat, outs[t][0].best_idx) == (sa.best_unsat, sa.best_idx)


def _agreement(cnf):
    """Fraction of literals true under the planted sigma; every clause's
    satisfaction under sigma and under its complement."""
    lits = np.asarray(cnf.lits)
    var = np.abs(lits) - 1
    true_sigma = (lits > 0) == (cnf.sigma[var] == 1)
    ptr = np.asarray(cnf.clause_ptr)
    sat_sigma = np.logical_or.reduceat(true_sigma, ptr[:-1])
    sat_comp = np.logical_or.reduceat(~true_sigma, ptr[:-1])
    return true_sigma.mean(), sat_sigma.all(), sat_comp.all()


def test_generator_planting_statistics():
    """naive planting makes a literal agree with sigma with
    probability 4/7 (3-SAT); 2-hidden planting (§8(f) f2) with probability
    1/2, and the complement of sigma satisfies every clause as well."""
    f1, s1, c1 = _agreement(planted_ksat(10_000, 42_000, 3, 1))
    assert s1 and not c1
    assert abs(f1 - 4 / 7) < 0.005
    f2, s2, c2 = _agreement(planted_ksat(10_000, 42_000, 3, 1, hidden=2))
    assert s2 and c2
    assert abs(f2 - 0.5) < 0.005
    # the naive instances are unchanged by the new option (same RNG stream)
    a, b = planted_ksat(50, 200, 3, 7), planted_ksat(50, 200, 3, 7, hidden=1)
    np.testing.assert_array_equal(a.lits, b.lits)
