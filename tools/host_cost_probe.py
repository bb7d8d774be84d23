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
    torch.cuda.set_device(0)
    comm = C.Comm.init_rank(1, C.unique_id(), 0)
    x = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    y = torch.zeros_like(x)
    h = comm.register(y)
    st = torch.cuda.current_stream()
    full = per_call(lambda: comm.alltoallv(x, [4096], [0], y, [4096], [0], st))
    U = ctypes.c_uint64 * 1
    args = (ctypes.c_void_p(x.data_ptr()), U(4096), U(0), ctypes.c_void_p(y.data_ptr()), U(4096), U(0), 0, comm._h,
            ctypes.c_void_p(st.cuda_stream))
    fn = _lib.lib().nimbleAlltoAllv
    raw = per_call(lambda: fn(*args))
    empty = per_call(lambda: torch.cuda._sleep(1))
    print(f"alltoallv via Python wrapper: {full:6.2f} us/call")
    print(f"alltoallv, prebuilt ctypes args: {raw:6.2f} us/call")
    print(f"one empty torch kernel launch: {empty:6.2f} us/call")
    comm.deregister(h)
    comm.destroy()


if __name__ == "__main__":
    main()
