"""Variant f2 "fp64 state" (SPEC S:278's choice; reading R30) in
the oracle: theta, m, v in fp64 and every rounding the fp32 readings
R13/R26/R27/R27b/R6 make is made to fp64 instead.  Pinned against fp64 torch
autograd of the dense formulation (element by element at 1e-12 relative,
floor 2^-48 x the magnitude of the summed terms), against fp64
torch.optim.AdamW (m, v to 1 ulp, theta to 1e-14 relative), against the
fp32 init (the fp64 Box-Muller value rounds to or_init's fp32 value), and
the Euler invariant of Eq. 5."""
import numpy as np
import pytest

from oracle import oracle as O
from test_oracle_pins2 import INSTANCES, _dense_grad64, _pt_abs, _torch_adamw64_step


def _check(ours, truth, terms, rtol=1e-12, floor=2.0 ** -48, what=""):
    err = np.abs(ours - truth)
    ok = err <= rtol * np.abs(truth) + floor * terms
    assert ok.all(), f"{what}: {np.count_nonzero(~ok)} elements off; worst {err[~ok].max()}"


def _advance(cnf, N, seed, steps, cfg):
    o = O.Oracle(cnf, N, seed, cfg=cfg)
    for _ in range(steps):
        o.step()
    return o


@pytest.mark.parametrize("name", sorted(INSTANCES))
@pytest.mark.parametrize("normalize,tau", [(1, 1.0), (1, 5.0), (0, 1.0), (3, 1.0)])
def test_fp64_gradient_vs_autograd(name, normalize, tau):
    cnf = O.binary_problem_matrix(INSTANCES[name]())
    for steps in (0, 9):
        o = _advance(cnf, 40, 2, steps, O.Config(normalize=normalize, tau=tau, state_fp64=1))
        assert o.theta.dtype == np.float64
        theta = o.theta.copy()
        s = o.step()
        assert s.grad.dtype == np.float64
        if normalize == 1 and (s.extra["guard"] != 0).any():
            continue
        truth = _dense_grad64(cnf, theta, tau, normalize)
        terms = _pt_abs(cnf, s.R, s.g) * np.abs(s.extra["rho"][:, None]) + np.abs(s.extra["cv"][:, None])
        _check(s.grad, truth, terms, what=f"{name} n{normalize} t{steps}")


def test_fp64_adamw_vs_torch():
    rng = np.random.default_rng(5)
    V, N = 5, 200
    theta = rng.standard_normal((V, N))
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    cfg = O.Config(state_fp64=1)
    L = O.lib()
    for t in list(range(0, 35)) + [59, 60, 99]:
        g = rng.standard_normal((V, N)) * 10.0 ** rng.uniform(-6, 2, size=(V, 1))
        lr = O.lr_at(t, cfg)
        th64, m64, v64 = _torch_adamw64_step(theta, m, v, g, lr, t + 1)
        th_prev, wdf = theta.copy(), 1 - lr * 1e-2
        L.or_adamw64(V, 0, N, O._p(theta), O._p(m), O._p(v), O._p(g), t, t + 1, lr, 0.9, 0.999, 1e-8, 1e-2, 0.0, 0)
        assert np.abs(m - m64).max() <= np.spacing(np.abs(m64)).max()
        assert (np.abs(v - v64) <= np.spacing(np.abs(v64))).all()
        # torch: (sqrt(v) / sqrt(bc2)) + eps and theta + (-lr/bc1) (m / den); the
        # canonical order (R6c) differs by a few ulps of the decayed theta and the step
        assert (np.abs(theta - th64) <= 1e-14 * (np.abs(th_prev * wdf) + np.abs(th64 - th_prev * wdf))).all(), t
        theta, m, v = th64.copy(), m64.copy(), v64.copy()


def test_fp64_init_rounds_to_fp32_init():
    V, N, seed = 37, 96, 0xABC
    o64 = O.Oracle(O.binary_problem_matrix(INSTANCES[sorted(INSTANCES)[0]]()), N, seed, cfg=O.Config(state_fp64=1))
    th32, _, _ = O.init_theta(o64.cnf.V, N, seed, 0, N)
    assert np.array_equal(o64.theta.astype(np.float32), th32)
    assert not np.array_equal(o64.theta, th32.astype(np.float64))      # genuinely fp64 values
    assert not o64.m.any() and not o64.v.any()


@pytest.mark.parametrize("normalize", [1, 3])
def test_fp64_euler_invariant(normalize):
    """Eq. 5 is scale invariant per row: sum_n theta dL/dtheta = 0 (guard inactive)."""
    cnf = O.binary_problem_matrix(INSTANCES[sorted(INSTANCES)[1]]())
    o = _advance(cnf, 64, 7, 4, O.Config(normalize=normalize, state_fp64=1))
    theta = o.theta.copy()
    s = o.step()
    for v in np.nonzero(s.extra["guard"] == 0)[0]:
        tot = float(np.sum(theta[v] * s.grad[v]))
        scale = float(np.sum(np.abs(theta[v] * s.grad[v]))) + 1e-300
        assert abs(tot) <= 1e-12 * scale
