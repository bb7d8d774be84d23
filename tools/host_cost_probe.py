"""Host cost of one alltoallv call, split into Python wrapper and C ABI (development aid, 1 GPU).

A 1-rank communicator exchanging a small self segment: the device work is a
few microseconds, so queueing many calls measures the host path alone.
"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import _lib  # noqa: E402
from paper_2604_00317_b200 import comm as C  # noqa: E402


def per_call(fn, n=2000):
    """Host microseconds per call (GPU work may lag behind; synchronized at the end)."""
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    return t * 1e6


def main():
    """1 rank by default; under torchrun, W ranks exchanging 4 KiB per pair."""
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        uid = [C.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, 0)
        comm = C.Comm.init_rank(world, uid[0], rank)
    else:
        comm = C.Comm.init_rank(1, C.unique_id(), 0)
    n = 4096
    x = torch.zeros(n * world, dtype=torch.uint8, device="cuda")
    y = torch.zeros_like(x)
    h = comm.register(y)
    st = torch.cuda.current_stream()
    counts, displs = [n] * world, [n * i for i in range(world)]
    full = per_call(lambda: comm.alltoallv(x, counts, displs, y, counts, displs, st))
    U = ctypes.c_uint64 * world
    args = (ctypes.c_void_p(x.data_ptr()), U(*counts), U(*displs), ctypes.c_void_p(y.data_ptr()), U(*counts),
            U(*displs), 0, comm._h, ctypes.c_void_p(st.cuda_stream))
    fn = _lib.lib().nimbleAlltoAllv
    raw = per_call(lambda: fn(*args))
    empty = per_call(lambda: torch.cuda._sleep(1))
    if rank == 0:
        print(f"W={world} alltoallv via Python wrapper: {full:6.2f} us/call")
        print(f"W={world} alltoallv, prebuilt ctypes args: {raw:6.2f} us/call")
        print(f"W={world} one empty torch kernel launch: {empty:6.2f} us/call")
    comm.deregister(h)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    comm.destroy()


if __name__ == "__main__":
    main()
