"""Pins of the oracle helpers that round 1 left unpinned, and element-wise
pins of the fp32 readings against fp64 ground truth.

* ``or_hist_stream``, ``or_backward_rows`` and ``oracle.step_sampled`` (the
  full-size parity helpers, tests/test_gpu_fullsize.py) are checked bit for bit
  against ``Oracle.step`` (itself pinned in test_oracle_pins.py) on uniform
  3-SAT, industrial K = 7, tautologies and repeated literals, at t = 0 and
  mid-trajectory (non-zero moments, an LR decay boundary, normalize 0/1/3).
* The fp32 readings R13 (J fixed point from fp32 products), R26 (fp32 g
  table), R27 (fp32 G chain), R27b (fp32 fused gradient) are checked ELEMENT
  BY ELEMENT against fp64 torch autograd of the dense formulation (PAPER.md
  Fig. 3, Eq. 1-5, l.189-191, l.226, l.262-269), and R6b/R6c (AdamW rounding)
  element by element against torch.optim.AdamW run in fp64
  (torch/optim/adam.py), both at the north star's 1e-5 relative tolerance.
  Stated absolute floor: 2^-20 times the magnitude of the terms the fp32
  value is formed from (|rho| sum_occ |dS/dR| + |c| for a gradient, |theta wdf| + |step|
  for a parameter, |m| + |g| for a moment) - 16 fp32 ulps of the operands,
  which only matters where the terms cancel.  Every element that needs the
  floor is one where |truth| < 5 % of the term magnitude (checked).
* The noise variate xi of reading R17 (``or_adamw``, sigma > 0) is pinned to
  its definition's distribution: uniform on [-1/2, 1/2) on the 2^-24 grid,
  independent across (candidate, variable, iteration), shard-invariant.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tsat_synth import Cnf, industrial_cnf, planted_ksat

FLOOR = 2.0 ** -20
RTOL = 1e-5


def _taut_dup_cnf():
    """Clauses with a tautology (x v ~x v y), repeated literals, a unit clause
    and long clauses (K = 7), on 24 variables."""
    rng = np.random.default_rng(5)
    cls = [[1, -1, 2], [3, 3, -4], [5, -6, 5, 7], [-8], [9, 10, 11, 12, 13, 14, 15]]
    for _ in range(90):
        k = int(rng.integers(2, 8))
        vs = rng.choice(24, size=k, replace=False) + 1
        cls.append([int(v) * (1 if rng.random() < 0.5 else -1) for v in vs])
    return Cnf.from_clauses(24, cls, name="taut-dup")


INSTANCES = {
    "uniform3": lambda: planted_ksat(60, 255, 3, 3),
    "industrial7": lambda: industrial_cnf(80, 330, 4),
    "taut_dup": _taut_dup_cnf,
}


def _advance(cnf, N, seed, steps, cfg):
    o = O.Oracle(cnf, N, seed, cfg=cfg)
    for _ in range(steps):
        o.step()
    return o


# ------------------------------------------------------------ full-size helpers
@pytest.mark.parametrize("name", sorted(INSTANCES))
def test_hist_stream_equals_histogram(name):
    """or_hist_stream (clause by clause, no C x N matrix) == or_histogram of
    or_clause_eval (§3.1.3-3.1.4)."""
    cnf = O.binary_problem_matrix(INSTANCES[name]())
    o = _advance(cnf, 96, 2, 3, O.Config())
    s = o.step()
    h = np.empty_like(s.h)
    rowbuf = np.empty(96, np.uint8)
    O.lib().or_hist_stream(cnf.C, O._p(cnf.clause_ptr), O._p(cnf.lits), 96, cnf.K, O._p(s.bits), O._p(h),
                           O._p(rowbuf))
    np.testing.assert_array_equal(h, s.h)


@pytest.mark.parametrize("name", sorted(INSTANCES))
def test_backward_rows_equals_backward(name):
    """or_backward_rows (per listed row, R recomputed clause by clause) ==
    or_backward (P^T fold over the stored R) for every row."""
    cnf = O.binary_problem_matrix(INSTANCES[name]())
    o = _advance(cnf, 64, 4, 2, O.Config())
    s = o.step()
    rows = np.arange(cnf.V, dtype=np.int32)[::-1].copy()       # every row, reversed order
    G = np.empty((cnf.V, 64))
    cnt = np.empty((64, cnf.K + 1), np.int32)
    rowbuf = np.empty(64, np.uint8)
    O.lib().or_backward_rows(cnf.C, O._p(cnf.clause_ptr), O._p(cnf.lits), 64, cnf.K, O._p(s.bits),
                             O._p(np.ascontiguousarray(s.g32)), O._p(rows), cnf.V, O._p(G), O._p(cnt), O._p(rowbuf))
    np.testing.assert_array_equal(G, s.G[rows])


@pytest.mark.parametrize("name", sorted(INSTANCES))
@pytest.mark.parametrize("normalize,t0", [(1, 0), (1, 31), (0, 5), (3, 29)])
def test_step_sampled_equals_oracle_step(name, normalize, t0):
    """oracle.step_sampled (the c3/c4 full-size parity reference) == Oracle.step:
    unsat, g32, S, loss and the sampled rows of theta, m, v, bit for bit."""
    cnf = INSTANCES[name]()
    cfg = O.Config(normalize=normalize)
    o = _advance(cnf, 64, 7, t0, cfg)
    th, m, v = o.theta.copy(), o.m.copy(), o.v.copy()
    rng = np.random.default_rng(t0 + 10 * normalize)
    rows = np.sort(rng.choice(cnf.V, size=min(17, cnf.V), replace=False)).astype(np.int32)
    unsat, g32, S, loss, th1, m1, v1 = O.step_sampled(cnf, th, m, v, t0, rows, cfg)
    s = o.step()
    np.testing.assert_array_equal(unsat, s.unsat)
    np.testing.assert_array_equal(g32, s.g32)
    np.testing.assert_array_equal(S, s.S)
    assert loss == s.loss
    np.testing.assert_array_equal(th1, o.theta[rows])
    np.testing.assert_array_equal(m1, o.m[rows])
    np.testing.assert_array_equal(v1, o.v[rows])


# ------------------------------------------------------------ element-wise fp32 readings
def _dense_grad64(cnf, theta, tau, normalize, eps=1e-8):
    """fp64 torch autograd of the paper's graph: Eq. 5 -> Eq. 2 (STE) -> Eq. 1
    (2V literal columns, A_neg = 1 - A_pos) -> Eq. 4 -> Eq. 3."""
    import torch
    V, N = theta.shape
    Pp = torch.zeros(cnf.C, V, dtype=torch.float64)
    Pn = torch.zeros(cnf.C, V, dtype=torch.float64)
    for c, cl in enumerate(cnf.clauses()):
        for x in cl:
            (Pp if x > 0 else Pn)[c, abs(x) - 1] = 1.0
    th = torch.tensor(theta.astype(np.float64), requires_grad=True)
    if normalize == 3:
        x = th / torch.clamp(th.abs().mean(dim=1, keepdim=True), min=eps)
    elif normalize:
        mu = th.mean(dim=1, keepdim=True)
        mag = torch.clamp(mu.abs(), min=eps)
        x = th / torch.where(mu >= 0, mag, -mag)
    else:
        x = th
    B = (x > 0).to(torch.float64)
    a = x + (B - x).detach()
    R = Pp @ a + Pn @ (1 - a)
    w = torch.exp(-tau * (R - R.detach().min(dim=0).values))
    S = (R * w).sum(0) / w.sum(0)
    L = -S.sum()
    L.backward()
    return th.grad.detach().numpy()


def _pt_abs(cnf, R, g):
    """sum over the occurrences of v of |dS_n/dR_cn|: the magnitude of the
    terms of the P^T sum that forms G_vn (numpy, fp64 table)."""
    out = np.zeros((cnf.V, R.shape[1]))
    cols = np.arange(R.shape[1])
    for c, cl in enumerate(cnf.clauses()):
        a = np.abs(g[cols, R[c]])
        for x in cl:
            out[abs(x) - 1] += a
    return out


def _check_elementwise(ours, truth, terms, what):
    err = np.abs(ours.astype(np.float64) - truth)
    ok = err <= RTOL * np.abs(truth) + FLOOR * terms
    assert ok.all(), f"{what}: {np.count_nonzero(~ok)} elements outside 1e-5 rel + floor; worst {err[~ok].max()}"
    needs_floor = err > RTOL * np.abs(truth)
    # the floor only ever serves cancellation: |truth| small against its terms
    assert (np.abs(truth[needs_floor]) < 0.05 * terms[needs_floor]).all(), what
    return int(needs_floor.sum())


@pytest.mark.parametrize("name", sorted(INSTANCES))
@pytest.mark.parametrize("normalize,tau", [(1, 1.0), (1, 0.5), (1, 5.0), (0, 1.0), (3, 1.0), (3, 2.0)])
def test_gradient_elementwise_vs_fp64_autograd(name, normalize, tau):
    """R26/R27/R27b/R13: the oracle's fp32 gradient dL/dtheta (STE backward +
    Eq. 5 Jacobian) agrees with fp64 autograd element by element within
    1e-5 relative (+ the stated floor), at t = 0 and after 12 iterations."""
    cnf = O.binary_problem_matrix(INSTANCES[name]())
    for steps in (0, 12):
        o = _advance(cnf, 48, 3, steps, O.Config(normalize=normalize, tau=tau))
        theta = o.theta.copy()
        s = o.step()
        if normalize == 1 and (s.extra["guard"] != 0).any():
            continue                                # guard rows: the clamp's derivative convention
        truth = _dense_grad64(cnf, theta, tau, normalize)
        terms = _pt_abs(cnf, s.R, s.g) * np.abs(s.extra["rho"][:, None]) + np.abs(s.extra["cv"][:, None])
        _check_elementwise(s.grad, truth, terms, f"{name} n{normalize} tau{tau} t{steps}")


def _torch_adamw64_step(theta, m, v, g, lr, step):
    """One torch.optim.AdamW step (PyTorch defaults, R6) in fp64 from the
    given fp32 state; returns (theta, m, v) in fp64."""
    import torch
    p = torch.nn.Parameter(torch.tensor(theta.astype(np.float64)))
    opt = torch.optim.AdamW([p], lr=lr, betas=(0.9, 0.999), eps=1e-8, weight_decay=1e-2, foreach=False)
    p.grad = torch.tensor(g.astype(np.float64))
    opt.step()                                  # creates the state (step 1)
    st = opt.state[p]
    with torch.no_grad():
        p.copy_(torch.tensor(theta.astype(np.float64)))
    st["exp_avg"].copy_(torch.tensor(m.astype(np.float64)))
    st["exp_avg_sq"].copy_(torch.tensor(v.astype(np.float64)))
    st["step"].fill_(float(step - 1))
    opt.step()
    return p.detach().numpy(), st["exp_avg"].numpy(), st["exp_avg_sq"].numpy()


def test_adamw_elementwise_vs_fp64_torch():
    """R6/R6b/R6c: each fp32 AdamW step of the oracle agrees with
    torch.optim.AdamW in fp64 from the same state, element by element, within
    1e-5 relative (+ floor), across LR decay boundaries and bias-correction
    steps 1..100, gradients over 8 decades."""
    rng = np.random.default_rng(11)
    V, N = 6, 256
    theta = rng.standard_normal((V, N)).astype(np.float32)
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    cfg = O.Config()
    L = O.lib()
    floors = 0
    for t in list(range(0, 40)) + [59, 60, 89, 99]:
        g = (rng.standard_normal((V, N)) * 10.0 ** rng.uniform(-6, 2, size=(V, 1))).astype(np.float32)
        lr = O.lr_at(t, cfg)
        th64, m64, v64 = _torch_adamw64_step(theta, m, v, g, lr, t + 1)
        wdf = 1 - lr * 1e-2
        th_terms = np.abs(theta.astype(np.float64) * wdf) + np.abs(th64 - theta.astype(np.float64) * wdf)
        m_terms = np.abs(m.astype(np.float64)) + np.abs(g.astype(np.float64))
        L.or_adamw(V, 0, N, O._p(theta), O._p(m), O._p(v), O._p(g), t, t + 1, lr, 0.9, 0.999, 1e-8, 1e-2, 0.0, 0)
        floors += _check_elementwise(theta, th64, th_terms, f"theta t{t}")
        floors += _check_elementwise(m, m64, m_terms, f"m t{t}")
        # v = beta2 v + (1 - beta2) g^2: no cancellation, pure relative
        np.testing.assert_array_less(np.abs(v - v64), RTOL * np.abs(v64) + 1e-300)
        # keep the state realistic: continue from torch's values rounded to fp32
        theta, m, v = th64.astype(np.float32), m64.astype(np.float32), v64.astype(np.float32)


# ------------------------------------------------------------ noise xi (R17)
def _xi(V, N, t, seed, n0=0, Nl=None):
    """xi recovered from or_adamw: theta = m = v = g = 0, wd = 0, sigma chosen
    so that nz = lr sigma = 2^-3, hence theta' = 2^-3 xi exactly."""
    Nl = N if Nl is None else Nl
    th = np.zeros((V, Nl), np.float32)
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    g = np.zeros_like(th)
    lr = 0.5
    O.lib().or_adamw(V, n0, Nl, O._p(th), O._p(m), O._p(v), O._p(g), t, t + 1, lr, 0.9, 0.999, 1e-8, 0.0, 0.25, seed)
    return th.astype(np.float64) * 8.0


def test_noise_xi_distribution():
    """R17: xi = (x >> 8) 2^-24 - 1/2 with x a Philox4x32-10 output (KAT-pinned
    in test_oracle_pins): uniform on [-1/2, 1/2) on the 2^-24 grid (KS test),
    mean 0, variance 1/12, uncorrelated between neighbouring candidates,
    variables and iterations; keyed by the global candidate (shard-invariant)
    and by the seed."""
    from scipy import stats
    V, N = 64, 1024
    a = _xi(V, N, 3, 0x1234)
    assert a.min() >= -0.5 and a.max() < 0.5
    k = (a + 0.5) * 2.0 ** 24
    assert np.array_equal(k, np.round(k))                   # on the 2^-24 grid
    x = a.ravel()
    assert stats.kstest(x + 0.5, "uniform").pvalue > 1e-3
    assert abs(x.mean()) < 4 * math.sqrt(1 / 12 / x.size)
    assert abs(x.var() - 1 / 12) < 0.01
    lim = 4 / math.sqrt(x.size)
    assert abs(np.corrcoef(a[:, 1:].ravel(), a[:, :-1].ravel())[0, 1]) < lim     # n, n+1
    assert abs(np.corrcoef(a[1:].ravel(), a[:-1].ravel())[0, 1]) < lim          # v, v+1
    b = _xi(V, N, 4, 0x1234)
    assert abs(np.corrcoef(a.ravel(), b.ravel())[0, 1]) < lim                    # t, t+1
    c = _xi(V, N, 3, 0x1235)
    assert abs(np.corrcoef(a.ravel(), c.ravel())[0, 1]) < lim                    # seed
    shard = _xi(V, N, 3, 0x1234, n0=384, Nl=128)
    np.testing.assert_array_equal(shard, a[:, 384:512])
    # xi is the documented function of the Philox output
    for (vv, n) in [(0, 0), (5, 7), (63, 1023)]:
        out = O.philox([n >> 2, vv, 1 + 3, 0], [0x1234, 0])
        assert a[vv, n] == float(out[n & 3] >> 8) * 2.0 ** -24 - 0.5


# ------------------------------------------------------------ OpenMP mode
def test_openmp_build_equals_single_thread():
    """SURVEY §8(c) "Form": the OpenMP build of the oracle (all host cores)
    gives the single-thread results bit for bit (disjoint-output loops, integer
    histograms), over several iterations of industrial K = 7 and the
    full-size helpers."""
    cnf = industrial_cnf(300, 1200, 9)
    ref = O.Oracle(cnf, 128, 3)
    outs = [ref.step() for _ in range(4)]
    try:
        O.use_openmp(True, threads=4)
        omp = O.Oracle(cnf, 128, 3)
        for s in outs:
            t = omp.step()
            np.testing.assert_array_equal(t.unsat, s.unsat)
            np.testing.assert_array_equal(t.G, s.G)
            assert t.loss == s.loss
        np.testing.assert_array_equal(omp.theta, ref.theta)
        np.testing.assert_array_equal(omp.m, ref.m)
        np.testing.assert_array_equal(omp.v, ref.v)
        rows = np.array([0, 7, 150], np.int32)
        a = O.step_sampled(cnf, ref.theta, ref.m, ref.v, 4, rows)
    finally:
        O.use_openmp(False)
    b = O.step_sampled(cnf, ref.theta, ref.m, ref.v, 4, rows)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x), np.asarray(y))


def test_tau_annealing_schedule():
    """Variant R29 (tau annealing): within each LR cycle tau_t goes
    geometrically from tau (t mod R = 0) to tau_final (t mod R = R - 1), with a
    constant ratio between consecutive iterations, and restarts with the LR
    (PAPER.md l.255-258); tau_final = 0 keeps Eq. 4's tau constant (R1)."""
    cfg = O.Config(tau=0.5, tau_final=8.0, restart_every=360)
    taus = np.array([O.tau_at(t, cfg) for t in range(720)])
    assert taus[0] == 0.5 and abs(taus[359] - 8.0) <= 1e-14 * 8.0
    assert np.array_equal(taus[:360], taus[360:])
    ratio = taus[1:360] / taus[:359]
    assert np.allclose(ratio, 16.0 ** (1 / 359), rtol=1e-13, atol=0)
    assert all(O.tau_at(t, O.Config(tau=2.0)) == 2.0 for t in range(0, 1000, 37))
    # the step uses the iteration's tau: one annealed step equals a constant-tau
    # step at that temperature
    from tsat_synth import planted_ksat
    cnf = planted_ksat(30, 120, 3, 4)
    o1 = O.Oracle(cnf, 32, 5, cfg=O.Config(tau=0.5, tau_final=8.0, restart_every=10))
    for _ in range(4):
        o1.step()
    t = o1.t
    o2 = O.Oracle(cnf, 32, 5, cfg=O.Config(tau=O.tau_at(t, o1.cfg), restart_every=10))
    o2.set_state(o1.theta, o1.m, o1.v, t)
    a, b = o1.step(), o2.step()
    assert np.array_equal(a.g32, b.g32) and np.array_equal(o1.theta, o2.theta)
