"""Multi-process host logic on CPU (gloo, world_size 2 and 8): the out-of-band
rendezvous nimbleCommInitRank uses, and bench.py's host-side helpers."""
import ctypes
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_00317_b200 import _lib
    from paper_2604_00317_b200 import comm as C
    uid = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    u = _lib.UniqueId()
    ctypes.memmove(ctypes.addressof(u), uid[0], 128)
    mine = (ctypes.c_uint64 * 3)(rank, rank * 1000 + 7, 0xABCDEF)
    out = (ctypes.c_uint64 * (3 * world))()
    rc = _lib.lib().nimbleBootstrapAllgather(ctypes.byref(u), rank, world, mine, 24, out)
    # bench.py helpers: per-rank matrix agreement and max-over-ranks timing
    import bench
    m = bench.workload_matrix(world, 1 << 20, 0.7)
    rows = [None] * world
    dist.all_gather_object(rows, m)
    t = bench.max_over_ranks(0.001 * (rank + 1))
    q.put((rank, rc, list(out), all(r == m for r in rows), t))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_bootstrap_and_host_helpers(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, rc, out, same, t in res:
        assert rc == 0
        assert out == [v for r in range(world) for v in (r, r * 1000 + 7, 0xABCDEF)]
        assert same
        assert t == pytest.approx(0.001 * world)


def test_bootstrap_rejects_foreign_id(lib):
    from paper_2604_00317_b200 import _lib
    u = _lib.UniqueId()
    out = (ctypes.c_uint64 * 2)()
    assert lib.nimbleBootstrapAllgather(ctypes.byref(u), 0, 1, out, 8, out) == 4
