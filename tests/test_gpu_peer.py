"""Peer-exchange multi-GPU path (tsat_create_peer): the
exchanges run inside the step kernels over peer memory.

This box has one GPU, so W = 2 runs as two ranks sharing it: two contexts in
one process (two host threads, each persistent k_update limited to part of
the SMs so both are resident), and two processes (CUDA IPC handles exchanged
over torch.distributed gloo).  Every case is compared bit for bit with the
oracle, which is shard-invariant (tests/test_oracle_pins.py)."""
import os
import threading

import numpy as np
import pytest

import oracle.oracle as O
from tsat_synth import industrial_cnf, planted_ksat

pytestmark = pytest.mark.gpu


def _cfg(ocfg):
    from paper_2511_07737_b200 import config_default
    c = config_default()
    for f in ("tau", "normalize", "beta1", "beta2", "eps", "weight_decay", "lr0", "lr_min", "decay_factor",
              "decay_every", "restart_every", "noise_sigma", "eps_norm", "reset_moments_on_restart", "tau_final"):
        setattr(c, f, getattr(ocfg, f))
    return c


def _pack(bits):
    V, N = bits.shape
    b = bits.reshape(V, N // 32, 32).astype(np.uint64)
    return (b << np.arange(32, dtype=np.uint64)).sum(axis=2).astype(np.uint32)


def _peer_solver(rank, world, stream=None):
    from paper_2511_07737_b200 import Solver
    return Solver(0, stream=stream, rank=rank, world=world, peer=True)


@pytest.mark.parametrize("case", ["c1", "industrial7", "ragged3", "c1-per-shard", "blk128", "blk256-ind", "blk512", "k15-256"])
def test_peer_w1_matches_oracle(case):
    """W = 1: the MODE 2 kernels exchanging with themselves reproduce the
    oracle bit for bit, step by step and through a multi-step graph."""
    ocfg = O.Config(normalize=2) if case == "c1-per-shard" else O.Config()
    if case.startswith("c1"):
        cnf, N = planted_ksat(20, 85, 3, 1), 64
    elif case == "industrial7":
        cnf, N = industrial_cnf(500, 2000, 4), 160
    elif case == "blk128":           # row-block kernel (MODE 2): 8 rows per warp, ragged tail
        cnf, N = planted_ksat(1003, 4213, 3, 5), 128
    elif case == "blk256-ind":
        cnf, N = industrial_cnf(701, 2800, 6), 256
    elif case == "k15-256":          # KB = 16 (all rows k_hub) through the peer row-block kernel
        from tsat_synth import coloring_cnf
        cnf, N = coloring_cnf(30, 15, 3, 4), 256
    elif case == "blk512":
        cnf, N = planted_ksat(777, 3263, 3, 8), 512
    else:
        cnf, N = planted_ksat(333, 1400, 3, 3), 96
    s = _peer_solver(0, 1)
    s.load_cnf(cnf)
    s.connect_peers()
    s.init_batch(N, 5, _cfg(ocfg))
    o = O.Oracle(cnf, N, 5, cfg=ocfg)
    th, m, v, _ = s.get_state()
    np.testing.assert_array_equal(th, o.theta)
    K = o.K
    KB = 4 if K <= 3 else (8 if K <= 7 else 16)
    for _ in range(12):
        info = s.step(1)
        ref = o.step()
        np.testing.assert_array_equal(s.query_unsat(), ref.unsat)
        np.testing.assert_array_equal(s.debug(3, np.uint32, (cnf.V, N // 32)), _pack(ref.bits))
        g = s.debug(1, np.float32, (KB, N))
        np.testing.assert_array_equal(g[:K + 1].T, ref.g32)
        th, m, v, _ = s.get_state()
        np.testing.assert_array_equal(th, o.theta)
        np.testing.assert_array_equal(m, o.m)
        np.testing.assert_array_equal(v, o.v)
        assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)
        assert abs(info.loss - ref.loss) <= 1e-9 * abs(ref.loss)
    info = s.step(17)
    for _ in range(17):
        ref = o.step()
    th, _, _, t = s.get_state()
    assert t == o.t
    np.testing.assert_array_equal(th, o.theta)
    assert (info.best_unsat, info.best_idx) == (ref.best_unsat, ref.best_idx)
    s.close()


def _run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    [t.start() for t in th]
    [t.join(timeout=600) for t in th]
    if errs:
        raise errs[0]


@pytest.mark.parametrize("normalize,N", [(1, 256), (2, 256), (3, 256), (1, 512), (1, 1024)])
def test_peer_two_ranks_one_gpu(normalize, N, monkeypatch):
    """W = 2 in one process: two contexts on their own streams, stepped from two
    host threads; the rank-concatenated state equals the oracle's (1 shard
    for normalize = 1 and 3; per-shard oracle ranks for normalize = 2)."""
    import torch
    monkeypatch.setenv("TSAT_UPD_GRID", "70")        # both persistent kernels resident on one GPU
    cnf = planted_ksat(400, 1680, 3, 7)
    W, seed = 2, 11              # N_l = N / 2: 128 and 256 run the row-block kernel, 512 the per-row one
    ocfg = O.Config(normalize=normalize)
    streams = [torch.cuda.Stream(0) for _ in range(W)]
    ss = [_peer_solver(r, W, stream=streams[r]) for r in range(W)]
    for s in ss:
        s.load_cnf(cnf)
    hs = [s.peer_handle() for s in ss]
    for s in ss:
        s.peer_open(hs)
    _run_threads([lambda s=s: s.init_batch(N, seed, _cfg(ocfg)) for s in ss])
    if normalize != 2:
        o = O.Oracle(cnf, N, seed, cfg=ocfg)
        refs = None
    else:
        import test_oracle_pins as P
        shards, _ = P.run_sharded(cnf, N, seed, W, 0, cfg=ocfg)
    infos = [None] * W
    for k in (1, 1, 6, 13):
        def go(r):
            infos[r] = ss[r].step(k)
        _run_threads([lambda r=r: go(r) for r in range(W)])
        if normalize != 2:
            for _ in range(k):
                refs = o.step()
            ref_theta = o.theta
            ref_unsat = refs.unsat
            best = (refs.best_unsat, refs.best_idx)
        else:
            outs = [None] * W
            import threading as _t
            comm = P.ThreadComm(W)
            for r, sh in enumerate(shards):
                sh.comm = comm.rank(r)

            def work(r):
                for _ in range(k):
                    outs[r] = shards[r].step()
            tt = [_t.Thread(target=work, args=(r,)) for r in range(W)]
            [x.start() for x in tt]
            [x.join() for x in tt]
            ref_theta = np.concatenate([sh.theta for sh in shards], axis=1)
            ref_unsat = np.concatenate([x.unsat for x in outs])
            best = (outs[0].best_unsat, outs[0].best_idx)
        th = np.concatenate([s.get_state()[0] for s in ss], axis=1)
        np.testing.assert_array_equal(th, ref_theta)
        un = np.concatenate([s.query_unsat() for s in ss])
        np.testing.assert_array_equal(un, ref_unsat)
        for r in range(W):
            assert (infos[r].best_unsat, infos[r].best_idx) == best
    for s in ss:
        s.close()


def _mp_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    os.environ["TSAT_UPD_GRID"] = "70"
    from paper_2511_07737_b200 import Solver
    cnf = planted_ksat(300, 1260, 3, 9)
    s = Solver(0, rank=rank, world=world, peer=True)
    s.load_cnf(cnf)
    s.connect_peers()
    s.init_batch(192, 3)
    info = s.step(9)
    th = s.get_state()[0]
    np.save(os.path.join(out_dir, f"theta{rank}.npy"), th)
    np.save(os.path.join(out_dir, f"info{rank}.npy"), np.array([info.best_unsat, info.best_idx, info.t]))
    s.close()
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_two_processes_ipc(tmp_path):
    """W = 2 as two processes on one GPU: exchange buffers mapped with CUDA IPC
    (handles all-gathered over gloo), 9 steps in one graph; equals the oracle."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(_mp_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    cnf = planted_ksat(300, 1260, 3, 9)
    o = O.Oracle(cnf, 192, 3)
    for _ in range(9):
        ref = o.step()
    th = np.concatenate([np.load(tmp_path / f"theta{r}.npy") for r in range(2)], axis=1)
    np.testing.assert_array_equal(th, o.theta)
    for r in range(2):
        bu, bi, t = np.load(tmp_path / f"info{r}.npy")
        assert (bu, bi, t) == (ref.best_unsat, ref.best_idx, 9)


def test_peer_export_is_global(monkeypatch):
    """tsat_export_best over W = 2 peer contexts is one collective: both ranks
    return the same M best candidates of the WHOLE batch, with the
    oracle's k most confident literals, although each rank holds
    only half of the candidates and only the owner reads a candidate's bits."""
    import torch
    monkeypatch.setenv("TSAT_UPD_GRID", "70")
    cnf = planted_ksat(400, 1680, 3, 21)
    N, W, seed, M = 256, 2, 13, 7
    streams = [torch.cuda.Stream(0) for _ in range(W)]
    ss = [_peer_solver(r, W, stream=streams[r]) for r in range(W)]
    for s in ss:
        s.load_cnf(cnf)
    hs = [s.peer_handle() for s in ss]
    for s in ss:
        s.peer_open(hs)
    _run_threads([lambda s=s: s.init_batch(N, seed) for s in ss])
    _run_threads([lambda s=s: s.step(5) for s in ss])
    o = O.Oracle(cnf, N, seed)
    for _ in range(5):
        ref = o.step()
    outs = [None] * W

    def ex(r):
        outs[r] = ss[r].export_best(M, 0)
    _run_threads([lambda r=r: ex(r) for r in range(W)])
    idx, u = O.select_top(ref.unsat, M)
    k = O.compute_k(cnf.V)
    owners = set()
    for r in range(W):
        assert len(outs[r]) == M
        for gi, n, un in zip(outs[r], idx, u):
            assert (gi["candidate"], gi["unsat"]) == (n, un)
            lits, mags = O.export_partial(np.abs(ref.G[:, n]), ref.bits[:, n], k)
            np.testing.assert_array_equal(gi["lits"], lits)
            np.testing.assert_array_equal(gi["abs_grad"], mags.astype(np.float32))
            owners.add(int(n) // (N // W))
    assert owners == {0, 1}                 # the selection spans both ranks
    for s in ss:
        s.close()
