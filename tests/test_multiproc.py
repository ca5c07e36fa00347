"""Multi-process (world size 2, gloo, CPU) tests of the candidate-sharded
path's host logic:

* the oracle run on 2 candidate shards, with its cross-candidate reductions
  done by torch.distributed all-reduces, is bit-identical to 1 shard (the
  exchange is exact: int64 sums and maxima);
* the global export merge (top-M by (unsat, index)) equals the single-rank one;
* the NCCL unique-id broadcast gives every rank the same id;
* the peer path's handle exchange (Solver.connect_peers) hands every rank all
  W exchange-buffer handles in rank order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class GlooComm:
    """Oracle communicator over torch.distributed (gloo)."""

    def sum_i64(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a, np.int64).copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    def max(self, x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return type(x)(t.item()) if not isinstance(x, np.floating) else x.__class__(t.item())

    def min_key(self, k):
        t = torch.tensor([k[0], k[1]], dtype=torch.int64)
        out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(out, t)
        return min((int(o[0]), int(o[1])) for o in out)

    def gather_f64(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a, np.float64).copy())
        out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(out, t)
        return np.concatenate([o.numpy() for o in out])


def _worker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        from tsat_synth import industrial_cnf, planted_ksat
        from paper_2511_07737_b200.binding import merge_keys
        out = {}
        for name, cnf, nz in (("planted", planted_ksat(80, 336, 3, 7), 1), ("industrial", industrial_cnf(150, 500, 5), 1),
                              ("planted-mag", planted_ksat(80, 336, 3, 7), 3)):
            N = 64
            Nl = N // world
            o = O.Oracle(cnf, N, 11, n0=rank * Nl, Nl=Nl, cfg=O.Config(normalize=nz))
            o.comm = GlooComm()
            unsat, losses, best = [], [], []
            for _ in range(steps):
                s = o.step()
                unsat.append(s.unsat.copy())
                losses.append(s.loss)
                best.append((s.best_unsat, s.best_idx))
            out[name] = dict(theta=o.theta, m=o.m, v=o.v, unsat=unsat, losses=losses, best=best)
            # export selection (tsat_export_best's host step): each rank's first
            # 3 keys (unsat << 32 | global index) all-gathered, merged by the
            # library's tsat_merge_keys
            idx, u = O.select_top(unsat[-1], 3, n0=rank * Nl)
            local = torch.tensor(((u.astype(np.int64) << 32) | idx).astype(np.int64))
            allk = [torch.zeros_like(local) for _ in range(world)]
            dist.all_gather(allk, local)
            keys = torch.cat(allk).numpy().astype(np.uint64)
            sel = merge_keys(keys, 3)
            out[name]["merged"] = [(int(k & 0xffffffff), int(k >> 32)) for k in sel]
        # NCCL unique-id broadcast (host logic of Solver.distributed)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        out["uid"] = obj[0]
        # peer-path handle exchange (host logic of Solver.connect_peers)
        from paper_2511_07737_b200.binding import Solver

        class _Stub:
            def __init__(self):
                self.world, self.rank, self.opened = world, rank, None

            def peer_handle(self):
                return bytes([rank + 1]) * 64

            def peer_open(self, hs):
                self.opened = list(hs)

        st = _Stub()
        Solver.connect_peers(st)
        out["peer_handles"] = st.opened
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_oracle_bit_identical(world):
    from oracle import oracle as O
    from tsat_synth import industrial_cnf, planted_ksat
    steps = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, q)) for r in range(world)]
    [p.start() for p in procs]
    res = dict(q.get(timeout=300) for _ in range(world))
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    for name, cnf, nz in (("planted", planted_ksat(80, 336, 3, 7), 1), ("industrial", industrial_cnf(150, 500, 5), 1),
                          ("planted-mag", planted_ksat(80, 336, 3, 7), 3)):      # R28 over gloo too
        ref = O.Oracle(cnf, 64, 11, cfg=O.Config(normalize=nz))
        refs = [ref.step() for _ in range(steps)]
        th = np.concatenate([res[r][name]["theta"] for r in range(world)], axis=1)
        np.testing.assert_array_equal(th, ref.theta)
        np.testing.assert_array_equal(np.concatenate([res[r][name]["m"] for r in range(world)], axis=1), ref.m)
        np.testing.assert_array_equal(np.concatenate([res[r][name]["v"] for r in range(world)], axis=1), ref.v)
        for t in range(steps):
            np.testing.assert_array_equal(np.concatenate([res[r][name]["unsat"][t] for r in range(world)]), refs[t].unsat)
            for r in range(world):
                assert res[r][name]["best"][t] == (refs[t].best_unsat, refs[t].best_idx)
                assert abs(res[r][name]["losses"][t] - refs[t].loss) <= 1e-12 * abs(refs[t].loss)
        idx, u = O.select_top(refs[-1].unsat, 3)
        for r in range(world):
            assert res[r][name]["merged"] == [(int(i), int(x)) for i, x in zip(idx, u)]
    assert res[0]["uid"] == res[1]["uid"] == bytes(range(128))
    for r in range(world):
        assert res[r]["peer_handles"] == [bytes([k + 1]) * 64 for k in range(world)]
