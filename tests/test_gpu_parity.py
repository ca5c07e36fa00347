"""GPU parity: the CUDA path (through the C-ABI / ctypes binding) against the
CPU oracle on identical seeded inputs.

Bar (BASELINE.json north_star): bit-exact unsat counts, binarised assignments
and SAT verdicts; floats within 1e-5 rel.  The canonical arithmetic
makes theta/m/v, the g table and S bit-exact too, so those are compared with
assert_array_equal; only the loss (a reduction whose order differs) uses a
tolerance (1e-12 rel).  Init uses libm vs CUDA transcendental functions:
<= 1 fp32 ulp and <= 1e-6 of the entries may differ.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tsat_synth import Cnf, coloring_cnf, enumeration_theta, fig1_cnf, industrial_cnf, make_config, planted_ksat, random_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_07737_b200 import build
    build.build()


def pack_bits(b):
    """V x N uint8 -> V x N/32 uint32 words (bit j of word w = candidate 32w+j)."""
    V, N = b.shape
    x = b.reshape(V, N // 32, 32).astype(np.uint64)
    return (x << np.arange(32, dtype=np.uint64)).sum(axis=2).astype(np.uint32)


def make_solver(sharded=False):
    from paper_2511_07737_b200 import Solver, nccl_unique_id
    if sharded:                     # candidate-sharded kernels + NCCL on a 1-rank communicator
        return Solver(0, rank=0, world=1, nccl_unique_id=nccl_unique_id())
    return Solver(0)


def make_pair(cnf, N, seed, cfg=None, state=None, t0=0, sharded=False):
    from paper_2511_07737_b200 import config_default
    s = make_solver(sharded)
    s.load_cnf(cnf)
    c = config_default()
    ocfg = cfg or O.Config()
    for f in ("tau", "normalize", "beta1", "beta2", "eps", "weight_decay", "lr0", "lr_min", "decay_factor",
              "decay_every", "restart_every", "noise_sigma", "eps_norm", "reset_moments_on_restart", "tau_final"):
        setattr(c, f, getattr(ocfg, f))
    s.init_batch(N, seed, c)
    o = O.Oracle(cnf, N, seed, cfg=ocfg)
    if state is not None:
        s.set_state(*state, t0)
        o.set_state(*state, t0)
    return s, o


def compare_step(s, o, cnf, what=""):
    info = s.step(1)
    ref = o.step()
    K = o.K
    KB = 4 if K <= 3 else (8 if K <= 7 else 16)
    N = ref.unsat.shape[0]
    unsat = s.query_unsat()
    np.testing.assert_array_equal(unsat, ref.unsat, err_msg=f"unsat {what} t={ref.t}")
    words = s.debug(3, np.uint32, (cnf.V, N // 32))
    np.testing.assert_array_equal(words, pack_bits(ref.bits), err_msg=f"bits {what} t={ref.t}")
    g = s.debug(1, np.float32, (KB, N))
    np.testing.assert_array_equal(g[:K + 1].T, ref.g32, err_msg=f"g {what} t={ref.t}")
    assert not g[K + 1:].any()
    S = s.debug(2, np.float64, (N,))
    np.testing.assert_array_equal(S, ref.S, err_msg=f"S {what} t={ref.t}")
    assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)
    assert abs(info.loss - ref.loss) <= 1e-12 * max(1.0, abs(ref.loss))
    th, m, v, t = s.get_state()
    assert t == o.t
    np.testing.assert_array_equal(th, o.theta, err_msg=f"theta {what} t={ref.t}")
    np.testing.assert_array_equal(m, o.m, err_msg=f"m {what} t={ref.t}")
    np.testing.assert_array_equal(v, o.v, err_msg=f"v {what} t={ref.t}")
    Q = s.debug(4, np.int64, (cnf.V,))
    Qo = np.empty(cnf.V, np.int64)
    rows = O.lib().or_row_sums_abs if o.cfg.normalize == 3 else O.lib().or_row_sums     # R28: sum |theta|
    rows(cnf.V, N, O._p(o.theta), O._p(Qo))
    np.testing.assert_array_equal(Q, Qo)
    return info, ref


def ulp_diff(a, b):
    ai = a.view(np.int32).astype(np.int64)
    bi = b.view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7fffffff), ai)
    bi = np.where(bi < 0, -(bi & 0x7fffffff), bi)
    return np.abs(ai - bi)


# ---------------------------------------------------------------- init
@pytest.mark.parametrize("V,N,seed", [(20, 64, 1), (1000, 4096, 7), (3, 32, 2**40 + 5)])
def test_init_matches_oracle(V, N, seed):
    cnf = planted_ksat(max(V, 3), 4 * max(V, 3), 3, 1)
    s, o = make_pair(cnf, N, seed)
    th, m, v, t = s.get_state()
    assert t == 0 and not m.any() and not v.any()
    d = ulp_diff(th, o.theta)
    assert d.max() <= 1
    assert (d > 0).mean() <= 1e-6


# ---------------------------------------------------------------- trajectories
def test_c1_trajectory_100_steps():
    """Config c1 (planted 3-SAT V=20, C=85, N=64): all 100 steps, every state."""
    cnf, cfg = make_config("c1")
    s, o = make_pair(cnf, cfg["N"], cfg["seed"])
    th, _, _, _ = s.get_state()
    if not np.array_equal(th, o.theta):      # libm/CUDA init ulp (see module doc): hand the
        s.set_state(o.theta, o.m, o.v, 0)      # ORACLE's theta0 to both sides
    for _ in range(100):
        compare_step(s, o, cnf, "c1")


@pytest.mark.parametrize("case", ["ragged3", "industrial7", "special", "two_sat"])
def test_ragged_and_mixed_instances(case):
    if case == "ragged3":
        cnf, N = planted_ksat(333, 1400, 3, 3), 96            # C not a multiple of the clause chunk, 3 words
    elif case == "industrial7":
        cnf, N = industrial_cnf(500, 2000, 4), 160            # K = 7, mixed lengths, hubs
    elif case == "special":
        base = planted_ksat(50, 200, 3, 9).clauses()
        base += [[1], [-2], [3, -3], [4, 4, -5], [6, 7, -6, 8]]   # units, tautologies, duplicate literal
        cnf, N = Cnf.from_clauses(50, base), 32
    else:
        cnf, N = planted_ksat(120, 200, 2, 5), 64
    state = random_state(cnf.V, N, seed=11)
    s, o = make_pair(cnf, N, 5, state=state, t0=0)
    for _ in range(12):
        compare_step(s, o, cnf, case)


def _uni3_with_hub(V=200, C=900, hub_occ=300, seed=4):
    """Uniform 3-SAT in which variable 1 occurs in hub_occ clauses (> 127 of
    one sign): a hub row of the uniform 3-SAT (plain-record) layout."""
    rng = np.random.default_rng(seed)
    cl = planted_ksat(V, C - hub_occ, 3, seed).clauses()
    for i in range(hub_occ):
        a, b = rng.choice(np.arange(2, V + 1), 2, replace=False)
        s1 = -1 if i % 3 else 1                   # 200 negated, 100 positive occurrences
        cl.append([s1 * 1, int(a) * (1 if rng.random() < .5 else -1), int(b) * (1 if rng.random() < .5 else -1)])
    return Cnf.from_clauses(V, cl)


@pytest.mark.parametrize("case", ["empty_clause", "no_clauses", "unused_vars", "uniform7", "k5_mixed", "uni3_hub"])
def test_degenerate_and_shape_cases(case):
    """Degenerate instances and layouts the bench configs do not reach: an
    empty clause (never satisfiable, R = 0 always), C = 0, variables without
    occurrences, uniform K = 7 (k_clause's uniform staging at K = 7), K = 5
    mixed lengths (KB = 8 with fewer bins live), and a uniform 3-SAT hub row."""
    if case == "empty_clause":
        cnf, N = Cnf.from_clauses(30, planted_ksat(30, 120, 3, 2).clauses() + [[]]), 64
    elif case == "no_clauses":
        cnf, N = Cnf.from_clauses(12, []), 32
    elif case == "unused_vars":
        cnf, N = Cnf.from_clauses(400, planted_ksat(100, 420, 3, 6).clauses()), 96
    elif case == "uniform7":
        cnf, N = planted_ksat(300, 1200, 7, 8), 128
    elif case == "k5_mixed":
        base = planted_ksat(200, 500, 3, 3).clauses() + planted_ksat(200, 300, 5, 4).clauses()
        cnf, N = Cnf.from_clauses(200, base), 64
    else:
        cnf, N = _uni3_with_hub(), 256
    state = random_state(cnf.V, N, seed=13)
    s, o = make_pair(cnf, N, 7, state=state, t0=0)
    for _ in range(6):
        compare_step(s, o, cnf, case)
    if case == "uni3_hub":
        assert s.info.n_hub_rows >= 1
    if case == "empty_clause":
        assert s.get_info().best_unsat >= 1 and s.get_solution() is None


@pytest.mark.parametrize("case", ["industrial7", "lengths_1_to_7", "uniform5", "two_three", "many_chunks", "industrial7_n2048"])
def test_length_segment_clause_eval(case):
    """k_clause_seg (>= 1024 candidates, every K <= 7 instance but uniform
    3-SAT): clauses regrouped by length, L gathers and L + 1 bins per clause,
    short (L <= 3) and long (L = 4..7) kernels.  Cases: the industrial mix with
    hubs; every length 1..7 plus an empty clause, a tautology and a duplicate
    literal (ragged segments); uniform K = 5 (one long segment); a 2-SAT +
    3-SAT mix (KB = 4: bin 3 derived, short kernel only); and enough clauses
    that every warp accumulates several chunks into the CTA fields.  The
    histograms are checked through unsat / g / S / theta, bit-exact."""
    if case == "industrial7":
        cnf, N = industrial_cnf(700, 2800, 22), 1024
    elif case == "lengths_1_to_7":
        rng = np.random.default_rng(5)
        base = []
        for L in range(1, 8):
            for _ in range(37 * L + 3):
                vs = rng.choice(np.arange(1, 241), L, replace=False)
                base.append([int(v) * (1 if rng.random() < .5 else -1) for v in vs])
        base += [[], [7, -7, 9], [11, 11, -12]]
        cnf, N = Cnf.from_clauses(240, base), 1024
    elif case == "uniform5":
        cnf, N = planted_ksat(300, 900, 5, 2), 2048
    elif case == "two_three":
        base = planted_ksat(400, 900, 3, 3).clauses() + planted_ksat(400, 500, 2, 4).clauses()
        cnf, N = Cnf.from_clauses(400, base), 1024
    elif case == "many_chunks":
        cnf, N = industrial_cnf(3000, 40000, 3), 1024
    else:                                                   # c4's shape class: the N = 2048 KB = 8 instantiation
        cnf, N = industrial_cnf(900, 3600, 12), 2048
    state = random_state(cnf.V, N, seed=19)
    s, o = make_pair(cnf, N, 3, state=state, t0=0)
    for _ in range(4):
        compare_step(s, o, cnf, case)


def test_uniform3_n1024_eight_plane_counters():
    """Uniform 3-SAT at N = 1024 with one variable in 40 negated clauses (> 31
    same-sign occurrences, < 128: not a hub) - the 8-plane counter path with
    the compile-time N = 1024 instantiation (c3's shape).  Bit-exact."""
    rng = np.random.default_rng(23)
    cl = planted_ksat(400, 1600, 3, 23).clauses()
    for i in range(40):
        a, b = rng.choice(np.arange(2, 401), 2, replace=False)
        cl.append([-1, int(a) * (1 if rng.random() < .5 else -1), int(b) * (1 if rng.random() < .5 else -1)])
    cnf, N = Cnf.from_clauses(400, cl), 1024
    state = random_state(cnf.V, N, seed=23)
    s, o = make_pair(cnf, N, 4, state=state, t0=0)
    assert s.info.n_hub_rows == 0
    for _ in range(4):
        compare_step(s, o, cnf, "uni3-n1024-cw8")


@pytest.mark.parametrize("N", [128, 256, 384, 512])
@pytest.mark.parametrize("kind", ["planted3", "industrial7"])
def test_row_block_kernel(kind, N):
    """Small shards (N < 1024, N % 128 == 0) run k_update_blk: a warp covers
    RB = 32 / (N/32) rows (8, 4, 2, 2 here), gathers all of them at once and
    streams the block's rows as one float4 stream.  V is not a multiple of RB
    (ragged last block); industrial7 has hub rows inside blocks and the
    batched-record layout (KB = 8).  k_clause splits its warps into
    sub-groups of N/32 lanes at these sizes.  Bit-exact against the oracle."""
    if kind == "planted3":
        cnf = planted_ksat(1003, 4213, 3, 21)
    else:
        cnf = industrial_cnf(701, 2800, 22)
    state = random_state(cnf.V, N, seed=17)
    s, o = make_pair(cnf, N, 9, state=state, t0=0)
    for _ in range(5):
        compare_step(s, o, cnf, f"{kind} N={N}")
    info = s.step(9)
    for _ in range(9):
        ref = o.step()
    th, m, v, _ = s.get_state()
    np.testing.assert_array_equal(th, o.theta)
    np.testing.assert_array_equal(v, o.v)
    assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)


@pytest.mark.parametrize("case", ["planted15_blk", "color15", "color9_mixed", "planted12_w1024", "color15_chunked"])
def test_long_clauses_k_gt_7(case):
    """clauses longer than 7 (KB = 16: 4-bit R, 15 counted bins,
    every row counted by k_hub in two 8-bin passes, k_clause_wide).  Planted
    15-SAT through the row-block kernel (N = 128), graph 15- and 9-colouring
    (at-least-one clauses of length 15 / 9 plus binary clauses; the shape of
    PAPER.md Table 1's 6g_6color) through the per-row kernel, a 1024-candidate
    batch, and the chunked large-batch sequence (g table 16 x 4 B x N > smem)."""
    if case == "planted15_blk":
        cnf, N = planted_ksat(301, 260, 15, 3), 128
    elif case == "color15":
        cnf, N = coloring_cnf(40, 15, 3, 1), 96
    elif case == "color9_mixed":
        base = coloring_cnf(30, 9, 4, 2).clauses() + planted_ksat(270, 300, 3, 4).clauses()
        cnf, N = Cnf.from_clauses(270, base), 160
    elif case == "planted12_w1024":
        cnf, N = planted_ksat(200, 180, 12, 5), 1024
    else:
        cnf, N = coloring_cnf(12, 15, 3, 3), 4096
    assert cnf.K > 7
    state = random_state(cnf.V, N, seed=19)
    s, o = make_pair(cnf, N, 3, state=state, t0=0)
    for _ in range(5):
        compare_step(s, o, cnf, case)
    if cnf.sigma is not None:                  # the planted model is a model (zero unsat on both sides)
        V = cnf.V
        th = np.where(cnf.sigma[:, None] > 0, 1.0, -1.0).astype(np.float32) * np.ones((V, N), np.float32)
        th[:, 1::2] *= -1.0                    # mean 0: guard active, d = +eps, bits = sign(theta)
        z = np.zeros_like(th)
        s.set_state(th, z, z, 0)
        o.set_state(th, z, z, 0)
        info, ref = compare_step(s, o, cnf, case + " planted model")
        assert ref.unsat[0] == 0 and info.best_unsat == 0


@pytest.mark.parametrize("case", ["planted3", "ragged", "k15_color", "k7_ind", "blk128"])
def test_dense_tensor_core_clause_eval(case):
    """config.clause_eval = 1 evaluates R = P A as a dense uint8
    tcgen05 product (k_dense.cu) and histograms R from TMEM; the whole step
    stays bit-exact against the oracle.  C not a multiple of the 128-clause
    tile, N not a multiple of the 256-candidate tile, 2V not a multiple of
    the 128-byte K chunk, K = 15 and K = 7 instances."""
    if case == "planted3":
        cnf, N = planted_ksat(256, 1075, 3, 2), 512
    elif case == "ragged":
        cnf, N = planted_ksat(173, 700, 3, 4), 96
    elif case == "k15_color":
        cnf, N = coloring_cnf(20, 15, 3, 5), 320
    elif case == "k7_ind":
        cnf, N = industrial_cnf(300, 1100, 6), 256
    else:
        cnf, N = planted_ksat(1003, 4213, 3, 21), 128
    state = random_state(cnf.V, N, seed=23)
    from paper_2511_07737_b200 import config_default
    s, o = make_pair(cnf, N, 4, state=state, t0=0)
    c = config_default()
    c.clause_eval = 1
    s.init_batch(N, 4, c)
    s.set_state(*state, 0)
    for _ in range(6):
        compare_step(s, o, cnf, f"dense {case}")


@pytest.mark.parametrize("kind", ["kb4_n8192", "kb8_n4096"])
def test_fused_g_table_in_l2(kind, monkeypatch):
    """Large per-GPU batches that still fit the fused kernel (BASELINE c5's
    8192-candidate share per GPU): the g table is read through L1 / L2 instead
    of shared memory so more warp groups fit.  Bit-exact against the oracle.
    (W = 1 runs these as cluster-split rows by default; the peer path, and
    TSAT_NO_CLUSTER here, keep this geometry.)"""
    monkeypatch.setenv("TSAT_NO_CLUSTER", "1")
    if kind == "kb4_n8192":
        cnf, N = planted_ksat(90, 380, 3, 3), 8192
    else:
        cnf, N = industrial_cnf(70, 260, 5), 4096
    state = random_state(cnf.V, N, seed=29)
    s, o = make_pair(cnf, N, 6, state=state, t0=0)
    for _ in range(4):
        compare_step(s, o, cnf, kind)


@pytest.mark.parametrize("case", ["planted3", "industrial7_mag", "k15", "reset_noise", "blk128"])
def test_fp64_state_variant(case):
    """SURVEY f2 / SPEC S:278: state_fp64 = 1 (reading R30): theta, m, v in
    fp64, the g table, G, the J terms, the gradient and AdamW in fp64, row
    sums in 128-bit fixed point at 2^-64 (k_fp64.cu).  Bit-exact against the
    oracle's fp64 path step by step (theta, m, v, bits, unsat, g32, best)."""
    from paper_2511_07737_b200 import config_default
    kw = {}
    if case == "planted3":
        cnf, N = planted_ksat(300, 1260, 3, 4), 512
    elif case == "industrial7_mag":
        cnf, N, kw = industrial_cnf(400, 1500, 5), 256, dict(normalize=3)
    elif case == "k15":
        cnf, N = coloring_cnf(15, 15, 3, 2), 288
    elif case == "reset_noise":
        cnf, N, kw = planted_ksat(200, 840, 3, 6), 320, dict(noise_sigma=0.2, reset_moments_on_restart=1,
                                                              restart_every=4, decay_every=2)
    else:
        cnf, N = planted_ksat(600, 2520, 3, 9), 128
    ocfg = O.Config(state_fp64=1, **kw)
    o = O.Oracle(cnf, N, 7, cfg=ocfg)
    c = config_default()
    for f in ("normalize", "noise_sigma", "reset_moments_on_restart", "restart_every", "decay_every"):
        setattr(c, f, getattr(ocfg, f))
    c.state_fp64 = 1
    from paper_2511_07737_b200 import Solver
    s = Solver(0)
    s.load_cnf(cnf)
    s.init_batch(N, 7, c)
    th, m, v, t = s.get_state()
    assert th.dtype == np.float64 and t == 0 and not m.any() and not v.any()
    d = np.abs(th - o.theta)
    # CUDA vs glibc fp64 log / sin / cos: a few ulps of the Box-Muller radius (absolute, since cos / sin
    # near their zeros have large relative error)
    assert (d <= 8 * np.spacing(1.0) * np.maximum(1.0, np.abs(o.theta))).all()
    s.set_state(o.theta, o.m, o.v, 0)
    K = o.K
    KB = 4 if K <= 3 else (8 if K <= 7 else 16)
    for step in range(7):
        info = s.step(1)
        ref = o.step()
        np.testing.assert_array_equal(s.query_unsat(), ref.unsat, err_msg=f"unsat {case} {step}")
        np.testing.assert_array_equal(s.debug(3, np.uint32, (cnf.V, N // 32)), pack_bits(ref.bits))
        g = s.debug(1, np.float32, (KB, N))
        np.testing.assert_array_equal(g[:K + 1].T, ref.g32)
        th, m, v, t = s.get_state()
        np.testing.assert_array_equal(th, o.theta, err_msg=f"theta {case} {step}")
        np.testing.assert_array_equal(m, o.m, err_msg=f"m {case} {step}")
        np.testing.assert_array_equal(v, o.v, err_msg=f"v {case} {step}")
        assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)
        assert abs(info.loss - ref.loss) <= 1e-12 * max(1.0, abs(ref.loss))
    info = s.step(9)
    for _ in range(9):
        ref = o.step()
    th, _, _, _ = s.get_state()
    np.testing.assert_array_equal(th, o.theta)
    ex = s.export_best(2)                       # |G| from the fp64 G of the evaluated state
    assert len(ex) == 2 and len(ex[0]["lits"]) == min(cnf.V, 20)


def test_fp64_state_fig1_solves():
    from paper_2511_07737_b200 import Solver, config_default
    c = config_default()
    c.state_fp64 = 1
    s = Solver(0)
    s.load_cnf(fig1_cnf())
    s.init_batch(32, 1, c)
    info = s.step(30)
    assert info.solved
    vals, idx, st = s.get_solution()
    assert tuple(vals) in {(1, 0, 0, 1), (1, 1, 0, 1)}
    import pytest as _p
    with _p.raises(Exception):
        s.set_state(np.zeros((4, 32), np.float32), np.zeros((4, 32), np.float32), np.zeros((4, 32), np.float32), 0)


def test_lr_boundaries_and_restart():
    """Cross the t = 29/30 decay and the t = 359/360 restart (R9)."""
    cnf = planted_ksat(200, 840, 3, 6)
    N = 128
    state = random_state(cnf.V, N, seed=3)
    for t0 in (27, 357):
        s, o = make_pair(cnf, N, 2, state=state, t0=t0)
        for _ in range(5):
            compare_step(s, o, cnf, f"t0={t0}")


@pytest.mark.parametrize("variant", [dict(normalize=0), dict(normalize=3), dict(weight_decay=0.0), dict(tau=5.0), dict(tau=0.5),
                                     dict(noise_sigma=0.3),
                                     dict(reset_moments_on_restart=1, restart_every=3, decay_every=2),
                                     dict(normalize=2), dict(tau=0.5, tau_final=8.0, restart_every=7, decay_every=3)])
def test_variants(variant):
    cnf = planted_ksat(150, 630, 3, 8)
    cfg = O.Config(**variant)
    s, o = make_pair(cnf, 96, 4, cfg=cfg)
    th, _, _, _ = s.get_state()
    s.set_state(o.theta, o.m, o.v, 0)
    for _ in range(8):
        compare_step(s, o, cnf, str(variant))


def test_multi_step_graph_launch_matches():
    """tsat_step(k) replays a k-iteration CUDA graph: same result as the oracle's k steps."""
    cnf = planted_ksat(400, 1680, 3, 12)
    N = 256
    s, o = make_pair(cnf, N, 21)
    s.set_state(o.theta, o.m, o.v, 0)
    for k in (10, 7, 33):
        info = s.step(k)
        for _ in range(k):
            ref = o.step()
        th, m, v, t = s.get_state()
        assert t == o.t
        np.testing.assert_array_equal(th, o.theta)
        np.testing.assert_array_equal(m, o.m)
        np.testing.assert_array_equal(v, o.v)
        np.testing.assert_array_equal(s.query_unsat(), ref.unsat)
        assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)


def test_async_steps_and_unsat_readback():
    """tsat_step(1, NULL) calls queue without draining the GPU (double-buffered
    step table) and tsat_query_unsat_async copies each step's counts into
    pinned memory read during the next step: the same counts and state as the
    oracle's step by step."""
    import torch
    cnf = planted_ksat(300, 1275, 3, 5)
    N = 128
    s, o = make_pair(cnf, N, 31)
    pins = [torch.empty(N, dtype=torch.int32, pin_memory=True) for _ in range(3)]
    for i in range(3):
        s.step(1, wait=False)
        s.query_unsat_async(pins[i].data_ptr())
    s.sync()
    for i in range(3):
        ref = o.step()
        np.testing.assert_array_equal(pins[i].numpy(), ref.unsat)
    th, m, v, t = s.get_state()
    assert t == o.t == 3
    np.testing.assert_array_equal(th, o.theta)
    np.testing.assert_array_equal(v, o.v)
    for _ in range(70):                       # many queued calls: the table slots alternate
        s.step(1, wait=False)
    for _ in range(70):
        ref = o.step()
    info = s.get_info()
    np.testing.assert_array_equal(s.query_unsat(), ref.unsat)
    assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)
    th, m, v, t = s.get_state()
    np.testing.assert_array_equal(th, o.theta)


def test_c2_full_size_two_steps():
    """Config c2 at full size (V=10k, C=42k, N=4096), bench's configuration."""
    cnf, cfg = make_config("c2")
    s, o = make_pair(cnf, cfg["N"], cfg["seed"])
    th, _, _, _ = s.get_state()
    d = ulp_diff(th, o.theta)
    assert d.max() <= 1 and (d > 0).mean() <= 1e-6
    s.set_state(o.theta, o.m, o.v, 0)
    for _ in range(2):
        compare_step(s, o, cnf, "c2")


# ---------------------------------------------------------------- forward pins at scale
def test_enumeration_all_assignments_v20():
    """Brute force: all 2^20 assignments of a planted 20-variable instance, in
    64 batches of 16384 (normalize off so theta's sign is the assignment);
    GPU unsat counts equal direct evaluation; min = 0 (the planted model)."""
    cnf = planted_ksat(20, 85, 3, 1)
    V, B = 20, 16384
    th = enumeration_theta(V)
    lits = np.array(cnf.clauses())
    var = np.abs(lits) - 1
    from paper_2511_07737_b200 import Solver, config_default
    s = Solver(0)
    s.load_cnf(cnf)
    c = config_default()
    c.normalize = 0
    s.init_batch(B, 1, c)
    allu = []
    for b in range(64):
        sl = th[:, b * B:(b + 1) * B]
        s.set_state(np.ascontiguousarray(sl), np.zeros_like(sl), np.zeros_like(sl), 0)
        s.step(1)
        allu.append(s.query_unsat().copy())
    unsat = np.concatenate(allu)
    n = np.arange(1 << V, dtype=np.int64)
    vals = ((n[None, None, :] >> var[:, :, None]) & 1) == (lits[:, :, None] > 0)
    ref = (~vals.any(axis=1)).sum(axis=0)
    np.testing.assert_array_equal(unsat, ref)
    assert unsat.min() == 0


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_properties(name):
    """Configs c3/c4/c5 at full size (c5: N = 65536 on one GPU, 26 GB of
    state, the chunked split sequence): init rows equal the oracle's; unsat
    counts equal direct evaluation of the exported model bits."""
    cnf, cfg = make_config(name)
    N = cfg["N"]
    from paper_2511_07737_b200 import Solver
    s = Solver(0)
    s.load_cnf(cnf)
    s.init_batch(N, cfg["seed"])
    rows = 64
    th0 = s.get_rows(np.arange(rows, dtype=np.int32))[0]
    ref, _, _ = O.init_theta(rows, N, cfg["seed"])
    assert ulp_diff(th0, ref).max() <= 1
    info = s.step(2)
    unsat = s.query_unsat()
    rng = np.random.default_rng(0)
    lits = cnf.lits
    var = np.abs(lits) - 1
    for n in rng.choice(N, 3, replace=False):
        b = s.export_model(int(n))
        val = np.where(lits > 0, b[var], 1 - b[var]).astype(np.int64)
        sat = np.add.reduceat(val, cnf.clause_ptr[:-1]) > 0
        assert unsat[n] == int((~sat).sum())
    assert info.best_unsat == unsat.min()


# ---------------------------------------------------------------- export / solution / resume
def test_export_matches_oracle():
    cnf = planted_ksat(300, 1260, 3, 14)
    N = 128
    s, o = make_pair(cnf, N, 3)
    s.set_state(o.theta, o.m, o.v, 0)
    for _ in range(6):
        s.step(1)
        ref = o.step()
    for k in (0, 7, 300):
        got = s.export_best(5, k)
        kk = O.compute_k(cnf.V) if k == 0 else k
        idx, u = O.select_top(ref.unsat, 5)
        for gi, n, un in zip(got, idx, u):
            assert (gi["candidate"], gi["unsat"]) == (n, un)
            lits, mags = O.export_partial(np.abs(ref.G[:, n]), ref.bits[:, n], kk)
            np.testing.assert_array_equal(gi["lits"], lits)
            np.testing.assert_array_equal(gi["abs_grad"], mags.astype(np.float32))
    for n in (0, 77, N - 1):
        np.testing.assert_array_equal(s.export_model(n), ref.bits[:, n])


def test_fig1_solution_and_verdict():
    cnf = fig1_cnf()
    s, o = make_pair(cnf, 32, 1)
    s.set_state(o.theta, o.m, o.v, 0)
    assert s.get_solution() is None
    for it in range(200):
        info = s.step(1)
        ref = o.step()
        assert info.best_unsat == ref.best_unsat
        if ref.best_unsat == 0:
            break
    assert info.solved and info.best_unsat == 0
    bits, idx, st = s.get_solution()
    assert (idx, st) == (ref.best_idx, ref.t)
    np.testing.assert_array_equal(bits, ref.bits[:, ref.best_idx])
    assert "".join(map(str, bits.tolist())) in ("1001", "1101")


def test_unsat_instance_never_solved():
    s, o = make_pair(Cnf.from_clauses(1, [[1], [-1]]), 64, 2)
    info = s.step(50)
    assert info.best_unsat == 1 and not info.solved and s.get_solution() is None


def test_checkpoint_resume_bit_exact():
    cnf = planted_ksat(250, 1050, 3, 15)
    from paper_2511_07737_b200 import Solver
    a = Solver(0); a.load_cnf(cnf); a.init_batch(256, 9)
    a.step(37)
    st = a.get_state()
    a.step(20)
    ref = a.get_state()
    b = Solver(0); b.load_cnf(cnf); b.init_batch(256, 9)
    b.set_state(st[0], st[1], st[2], st[3])
    b.step(20)
    got = b.get_state()
    for x, y in zip(got[:3], ref[:3]):
        np.testing.assert_array_equal(x, y)
    assert got[3] == ref[3] == 57


def test_determinism_two_runs():
    cnf = planted_ksat(500, 2100, 3, 16)
    from paper_2511_07737_b200 import Solver
    outs = []
    for _ in range(2):
        s = Solver(0); s.load_cnf(cnf); s.init_batch(512, 3)
        info = s.step(40)
        outs.append((s.get_state()[0], s.query_unsat().copy(), info.loss))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_error_paths():
    from paper_2511_07737_b200 import Solver, TsatError
    s = Solver(0)
    with pytest.raises(TsatError) as e:
        s.step(1)
    assert e.value.name == "TSAT_E_STATE"
    s.load_cnf(planted_ksat(30, 120, 3, 1))
    with pytest.raises(TsatError) as e:
        s.init_batch(48, 1)                      # N % 32 != 0
    assert e.value.name == "TSAT_E_ARG"
    s.init_batch(64, 1)
    with pytest.raises(TsatError) as e:
        s.query_unsat()                          # nothing evaluated yet
    assert e.value.name == "TSAT_E_STATE"
    with pytest.raises(TsatError) as e:
        s.step(0)
    assert e.value.name == "TSAT_E_ARG"


# ---------------------------------------------------------------- sharded path (1-rank NCCL communicator)
@pytest.mark.parametrize("case", ["c1", "industrial7", "ragged3", "c1-per-shard", "ragged3-reset", "industrial7-mag"])
def test_sharded_path_matches_oracle(case):
    """The multi-GPU kernels (phase A -> SUM J -> phase B -> SUM Q -> rows
    finish, plus the MAX exchange) on a 1-rank communicator reproduce the
    oracle bit for bit; also with the f2 variants (per-shard
    normalisation: no J/Q exchange; moment reset at LR restarts)."""
    cfg = None
    if case == "c1-per-shard":
        case, cfg = "c1", O.Config(normalize=2)
    elif case == "ragged3-reset":
        case, cfg = "ragged3", O.Config(reset_moments_on_restart=1, restart_every=7, decay_every=3)
    elif case == "industrial7-mag":
        case, cfg = "industrial7", O.Config(normalize=3)
    if case == "c1":
        cnf, N = planted_ksat(20, 85, 3, 1), 64
    elif case == "industrial7":
        cnf, N = industrial_cnf(500, 2000, 4), 160
    else:
        cnf, N = planted_ksat(333, 1400, 3, 3), 96
    s, o = make_pair(cnf, N, 5, cfg=cfg, sharded=True)
    th, _, _, _ = s.get_state()
    if not np.array_equal(th, o.theta):
        s.set_state(o.theta, o.m, o.v, 0)
    for _ in range(15):
        compare_step(s, o, cnf, "sharded-" + case)
    info = s.step(20)
    for _ in range(20):
        ref = o.step()
    th, m, v, t = s.get_state()
    np.testing.assert_array_equal(th, o.theta)
    assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)
    assert abs(info.loss - ref.loss) <= 1e-9 * abs(ref.loss)


def test_sharded_equals_fused_c2():
    """Sharded (W = 1 communicator) and fused single-GPU paths give identical
    states on config c2 (both are the canonical arithmetic)."""
    cnf, cfg = make_config("c2")
    a = make_solver(False); a.load_cnf(cnf); a.init_batch(cfg["N"], 3)
    b = make_solver(True); b.load_cnf(cnf); b.init_batch(cfg["N"], 3)
    ia, ib = a.step(12), b.step(12)
    for x, y in zip(a.get_state()[:3], b.get_state()[:3]):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(a.query_unsat(), b.query_unsat())
    assert (ia.best_unsat, ia.best_idx) == (ib.best_unsat, ib.best_idx)


# ---------------------------------------------------------------- cluster-split rows
@pytest.mark.parametrize("case", ["kb4_n8192", "kb4_n16384_noise", "kb8_hubs", "kb4_ragged_mag", "kb4_n65536"])
def test_cluster_split_rows(case, monkeypatch):
    """Large W = 1 batches (the g table of N candidates would leave fewer than
    4 warp groups): k_update MODE 3 splits every row's candidates over the CL
    CTAs of a thread-block cluster, each holding its slice of the g table in
    shared memory, and sums the row's exact int64 J and Q partials over DSMEM.
    Cases: CL = 2 (BASELINE c5's 8192 per GPU), CL = 4 with update noise, KB =
    8 with hub rows (industrial, N = 4096), a slice that is not a power of two
    (17408 = 4 x 4352) under normalize 3 (R28), and CL = 16 (c5's 65 536 on
    one GPU, non-portable cluster size).  Bit-exact against the oracle.
    (Opt-in, TSAT_CLUSTER=1: measured slower than the default geometries.)"""
    monkeypatch.setenv("TSAT_CLUSTER", "1")
    cfg = None
    if case == "kb4_n8192":
        cnf, N, cl = planted_ksat(90, 380, 3, 3), 8192, 2
    elif case == "kb4_n16384_noise":
        cnf, N, cl, cfg = planted_ksat(60, 250, 3, 2), 16384, 4, O.Config(noise_sigma=0.05)
    elif case == "kb8_hubs":
        cnf, N, cl = industrial_cnf(300, 1800, 8), 4096, 2
    elif case == "kb4_ragged_mag":
        cnf, N, cl, cfg = planted_ksat(70, 290, 3, 5), 17408, 4, O.Config(normalize=3)
    else:
        cnf, N, cl = planted_ksat(24, 100, 3, 4), 65536, 16
    state = random_state(cnf.V, N, seed=31)
    s, o = make_pair(cnf, N, 8, cfg=cfg, state=state, t0=0)
    g = s.update_geometry()
    assert g["cluster"] == cl and g["slice"] == N // cl, g
    for _ in range(3):
        compare_step(s, o, cnf, case)
    if case == "kb8_hubs":
        assert s.info.n_hub_rows >= 1
    info = s.step(4)
    for _ in range(4):
        ref = o.step()
    th, m, v, _ = s.get_state()
    np.testing.assert_array_equal(th, o.theta)
    np.testing.assert_array_equal(v, o.v)
    assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)


# ---------------------------------------------------------------- other code paths
@pytest.mark.parametrize("kind", ["kb4", "kb8", "kb4-ragged"])
def test_chunked_large_batch_path(kind, monkeypatch):
    """Batches too large for the fused kernel's shared memory (the g table of
    N candidates) run the split sequence with k_update work items of 4096
    (KB = 8: 2048) candidates, the g table read from L2 and exact int64 J
    atomics; same canonical results (also with a ragged last chunk).  (At W = 1
    these sizes run cluster-split rows by default; TSAT_NO_CLUSTER keeps the
    split sequence, which multi-GPU NCCL runs and unsplittable N still use.)"""
    monkeypatch.setenv("TSAT_NO_CLUSTER", "1")
    if kind == "kb4":
        cnf, N = planted_ksat(60, 250, 3, 2), 16384        # g table 256 KB > smem: 4 chunks
    elif kind == "kb8":
        cnf, N = industrial_cnf(80, 300, 6), 8192          # KB = 8: 256 KB, 4 chunks
    else:
        cnf, N = planted_ksat(70, 290, 3, 5), 17408        # 4 x 4096 + 1024
    s, o = make_pair(cnf, N, 3)
    base = 3 if cnf.V else 0
    assert s.kernels_per_step() >= base + 3               # update B, rows finish, step end
    assert s.update_geometry()["cluster"] == 0
    s.set_state(o.theta, o.m, o.v, 0)
    for _ in range(4):
        compare_step(s, o, cnf, "chunked-" + kind)
    info = s.step(5)
    for _ in range(5):
        ref = o.step()
    th, m, v, _ = s.get_state()
    np.testing.assert_array_equal(th, o.theta)
    np.testing.assert_array_equal(v, o.v)
    assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)


def test_hub_rows_parity_and_export():
    """An industrial-shaped instance with hub variables (k_hub pre-pass, split
    occurrence lists, int32 counts): bit-exact steps and export."""
    cnf = industrial_cnf(1500, 9000, 8)
    N = 192
    s, o = make_pair(cnf, N, 4)
    assert s.info.n_hub_rows > 0
    s.set_state(o.theta, o.m, o.v, 0)
    for _ in range(6):
        _, ref = compare_step(s, o, cnf, "hubs")
    got = s.export_best(3, 0)
    idx, u = O.select_top(ref.unsat, 3)
    k = O.compute_k(cnf.V)
    for gi, n, un in zip(got, idx, u):
        assert (gi["candidate"], gi["unsat"]) == (n, un)
        lits, mags = O.export_partial(np.abs(ref.G[:, n]), ref.bits[:, n], k)
        np.testing.assert_array_equal(gi["lits"], lits)
        np.testing.assert_array_equal(gi["abs_grad"], mags.astype(np.float32))


# ---------------------------------------------------------------- boundary (round 2)
def test_load_dimacs_equals_load_clauses():
    """tsat_load_dimacs on a context (SPEC S:41-49 parsing, dedup) gives the
    same CNF as tsat_load_clauses: identical steps, bit for bit, also against
    the oracle; the info block reports the parse (tautology, duplicates)."""
    from paper_2511_07737_b200 import Solver
    from tsat_synth import to_dimacs
    base = industrial_cnf(400, 1500, 12)
    cls = base.clauses() + [[3, -3, 5], [7, 7, -9]]
    cnf = Cnf.from_clauses(base.V, cls)
    text = b"c round-2 boundary test\n" + to_dimacs(cnf)
    a, b = Solver(0), Solver(0)
    ia = a.load_dimacs(text)
    ib = b.load_cnf(cnf)
    assert (ia.V, ia.C, ia.nnz, ia.K) == (ib.V, ib.C, ib.nnz, ib.K)
    assert ia.n_tautologies == ib.n_tautologies >= 1 and ia.n_duplicates == ib.n_duplicates == 1
    assert ia.header_C == cnf.C and ib.header_C == -1
    N = 96
    a.init_batch(N, 4)
    b.init_batch(N, 4)
    o = O.Oracle(cnf, N, 4)
    a.set_state(o.theta, o.m, o.v, 0)
    b.set_state(o.theta, o.m, o.v, 0)
    for _ in range(4):
        ia_, ib_ = a.step(1), b.step(1)
        ref = o.step()
        np.testing.assert_array_equal(a.query_unsat(), ref.unsat)
        np.testing.assert_array_equal(b.query_unsat(), ref.unsat)
        assert (ia_.best_unsat, ia_.best_idx) == (ib_.best_unsat, ib_.best_idx) == (ref.best_unsat, ref.best_idx)
    np.testing.assert_array_equal(a.get_state()[0], o.theta)
    np.testing.assert_array_equal(b.get_state()[0], o.theta)


def test_abi_size_checks():
    """host arrays of the wrong size are rejected (TSAT_E_ARG), not
    read out of bounds; a checkpoint of another batch size cannot be loaded."""
    from paper_2511_07737_b200 import TsatError
    from paper_2511_07737_b200.binding import _ptr
    import ctypes as ct
    cnf = planted_ksat(50, 210, 3, 2)
    s, o = make_pair(cnf, 64, 1)
    s.step(1)
    with pytest.raises(ValueError):
        s.set_state(o.theta[:, :32], o.m[:, :32], o.v[:, :32], 0)
    small = np.zeros(10, np.int32)
    first = ct.c_int64()
    assert s.lib.tsat_query_unsat(s.h, _ptr(small), small.size, ct.byref(first)) == 1
    th = np.zeros((50, 32), np.float32)
    assert s.lib.tsat_set_state(s.h, _ptr(th), _ptr(th), _ptr(th), th.size, 0) == 1
    assert s.lib.tsat_get_state(s.h, _ptr(th), None, None, th.size, None) == 1
    with pytest.raises(TsatError):
        s.export_best(64 + 1, 0)               # M > N_global


def test_export_sharded_path_matches_oracle():
    """The candidate-sharded (NCCL) path's export on a 1-rank communicator:
    the all-gather + library merge give the oracle's selection and literals."""
    cnf = planted_ksat(300, 1260, 3, 15)
    N = 128
    s, o = make_pair(cnf, N, 5, sharded=True)
    s.set_state(o.theta, o.m, o.v, 0)
    for _ in range(5):
        s.step(1)
        ref = o.step()
    got = s.export_best(4, 0)
    idx, u = O.select_top(ref.unsat, 4)
    k = O.compute_k(cnf.V)
    for gi, n, un in zip(got, idx, u):
        assert (gi["candidate"], gi["unsat"]) == (n, un)
        lits, mags = O.export_partial(np.abs(ref.G[:, n]), ref.bits[:, n], k)
        np.testing.assert_array_equal(gi["lits"], lits)
        np.testing.assert_array_equal(gi["abs_grad"], mags.astype(np.float32))
