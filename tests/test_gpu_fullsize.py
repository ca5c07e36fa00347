"""Parity at BASELINE.json's full sizes (configs c3, c4), one iteration in the
bench's launch configuration, on outputs the oracle can compute one by one:
every candidate's unsat count (the whole histogram is streamed clause by
clause), the g table and S of every candidate, the loss, and the updated
theta / m / v of sampled variable rows (including hub rows at c4).  The
oracle generates theta0, which both sides take as input."""
import numpy as np
import pytest

from oracle import oracle as O
from tsat_synth import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_07737_b200 import build
    build.build()


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_size_sampled_parity(name):
    from paper_2511_07737_b200 import Solver
    cnf, cfg = make_config(name)
    N = cfg["N"]
    th, m, v = O.init_theta(cnf.V, N, cfg["seed"])
    s = Solver(0)
    info = s.load_cnf(cnf)
    s.init_batch(N, cfg["seed"])
    s.set_state(th, m, v, 0)
    step = s.step(1)
    rng = np.random.default_rng(1)
    occ = np.bincount(np.abs(cnf.lits.astype(np.int64)) - 1, minlength=cnf.V)
    rows = np.unique(np.concatenate([rng.choice(cnf.V, 40, replace=False), np.argsort(-occ)[:8]])).astype(np.int32)
    unsat, g32, S, loss, th1, m1, v1 = O.step_sampled(cnf, th, m, v, 0, rows)
    del th, m, v
    np.testing.assert_array_equal(s.query_unsat(), unsat)
    K = O.binary_problem_matrix(cnf).K
    KB = 4 if K <= 3 else (8 if K <= 7 else 16)
    g = s.debug(1, np.float32, (KB, N))
    np.testing.assert_array_equal(g[:K + 1].T, g32)
    np.testing.assert_array_equal(s.debug(2, np.float64, (N,)), S)
    assert abs(step.loss - loss) <= 1e-12 * abs(loss)
    gth, gm, gv = s.get_rows(rows)
    np.testing.assert_array_equal(gth, th1)
    np.testing.assert_array_equal(gm, m1)
    np.testing.assert_array_equal(gv, v1)
    if name == "c4":
        assert info.n_hub_rows > 0
