"""Multi-process host logic of the N>1 path on CPU (gloo, world size 2 and 4):
the library's y-strip plan (hom2d_strip_plan, host-only C code) drives a halo
exchange that mirrors the NCCL message order of hom2d_api.cu; every rank must
receive exactly the global neighbour rows (periodic wrap / none at a
transmissive boundary).  Also the bench plumbing: NCCL-id broadcast and the
max-over-ranks timing reduction."""
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


def _global(nx, ny, npe):
    """canonical SoA state whose values encode (component, row, column, point)"""
    c, j, i, p = np.meshgrid(np.arange(4), np.arange(ny), np.arange(nx), np.arange(npe), indexing="ij")
    return (c * 1e6 + j * 1e3 + i * 1e1 + p * 1e-2).astype(np.float64)  # [c][j][i][p]


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1709_01619_b200 as P
    try:
        for method, k, bc in cases:
            nx, ny = 6, 4 * world
            cfg = P.make_config(nx, ny, method=method, k=k, bc=bc)
            plan = P.strip_plan(cfg, rank, world)
            npe = 1 if method == "fv" else (k + 1) ** 2
            glob = _global(nx, ny, npe)
            local = glob[:, plan.row0:plan.row0 + plan.nrows]
            G = plan.ghost_rows
            assert plan.row_values == nx * npe
            lo = np.zeros((4, G, nx, npe))
            hi = np.zeros((4, G, nx, npe))
            # same per-peer message order as hom2d_api.cu exchange()
            for c in range(4):
                reqs = []
                if plan.has_hi:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(local[c, -G:])), plan.peer_hi))
                if plan.has_lo:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(local[c, :G])), plan.peer_lo))
                tlo = torch.zeros(G, nx, npe, dtype=torch.float64)
                thi = torch.zeros(G, nx, npe, dtype=torch.float64)
                if plan.has_lo:
                    dist.recv(tlo, plan.peer_lo)
                if plan.has_hi:
                    dist.recv(thi, plan.peer_hi)
                for r in reqs:
                    r.wait()
                lo[c], hi[c] = tlo.numpy(), thi.numpy()
            # expected ghost rows
            rows_lo = [(plan.row0 - G + g) for g in range(G)]
            rows_hi = [(plan.row0 + plan.nrows + g) for g in range(G)]
            if plan.has_lo:
                np.testing.assert_array_equal(lo, glob[:, [r % ny for r in rows_lo]])
            else:
                assert bc == 1 and rank == 0
            if plan.has_hi:
                np.testing.assert_array_equal(hi, glob[:, [r % ny for r in rows_hi]])
            else:
                assert bc == 1 and rank == world - 1
        # bench plumbing: id broadcast, max over ranks
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_strip_exchange_gloo(world):
    from paper_1709_01619_b200 import build
    build.build()
    cases = [("cpr", 3, 0), ("cpr", 2, 1), ("fv", 1, 0), ("fv", 2, 1), ("dg", 1, 0)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def test_strip_plan_covers_grid():
    import paper_1709_01619_b200 as P
    for world in (1, 2, 4, 8):
        cfg = P.make_config(16, 64, method="cpr", k=3)
        plans = [P.strip_plan(cfg, r, world) for r in range(world)]
        assert [p.row0 for p in plans] == [r * 64 // world for r in range(world)]
        assert sum(p.nrows for p in plans) == 64
        for r, p in enumerate(plans):
            assert p.peer_hi == (r + 1) % world and p.peer_lo == (r - 1) % world
    with pytest.raises(P.Hom2dError):
        P.strip_plan(P.make_config(16, 10, method="cpr", k=3), 0, 4)   # ny % nranks != 0
    with pytest.raises(P.Hom2dError):
        P.strip_plan(P.make_config(16, 8, method="fv", k=1), 0, 8)     # FV needs 2 ghost rows


class _FakeSolver:
    """stands in for Solver in connect_peers: ids are bytes naming the rank"""
    def __init__(self, rank):
        self.rank = rank
        self.got = None

    def peer_id(self):
        return b"rank%03d" % self.rank + bytes(73)

    def peer_connect(self, lo, hi):
        self.got = (lo, hi)


def _peer_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1709_01619_b200 as P
    try:
        s = _FakeSolver(rank)
        ids = P.connect_peers(s)
        assert [i[:7] for i in ids] == [b"rank%03d" % r for r in range(world)]
        lo, hi = s.got
        # the strip neighbours of hom2d_strip_plan (periodic in y)
        plan = P.strip_plan(P.make_config(6, 4 * world), rank, world)
        assert lo[:7] == b"rank%03d" % plan.peer_lo and hi[:7] == b"rank%03d" % plan.peer_hi
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_id_exchange_gloo(world):
    """The peer-memory halo's host plumbing (connect_peers): every rank gets all
    ids by all_gather and connects to the ids of its strip-plan neighbours."""
    from paper_1709_01619_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
