"""Host cost of scheduling one rank's work for a new matrix (CPU only).

  cuts  -- build_schedule: the rank's flows (what a communicator does per new
           matrix; the device generator merges them, gen_items_kernel)
  merge -- the same plus the host merge into the item list (what round 1 did,
           and what nimbleDebugSchedule still returns)
Plan: nimblePlanCreate on the nvswitch model (the comm uses the direct plan
there, which this upper-bounds)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import _lib  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

lib = _lib.lib()


def per_call(fn, k=50):
    fn()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    return (time.perf_counter() - t0) / k * 1e6


for R, per in ((8, 256 << 20), (8, 16 << 20), (4, 256 << 20)):
    topo = P.build_canonical(1, R, 0, 900e9, 0, P.NVSWITCH)
    m = P.gen_skewed_a2av(R, per, 0.7, 0)
    off = [0 if i // R == i % R else v for i, v in enumerate(m)]
    cfg = P.PlannerConfig().to_c()
    h = ctypes.c_void_p()
    plan_us = per_call(lambda: (lib.nimblePlanCreate(topo.handle, R, R, _lib.u64_array(off), ctypes.byref(cfg),
                                                     ctypes.byref(h)), lib.nimblePlanDestroy(h)))
    _lib.call("nimblePlanCreate", topo.handle, R, R, _lib.u64_array(off), ctypes.byref(cfg), ctypes.byref(h))
    n = ctypes.c_int()
    for rank in (0, 1):
        args = (h, rank, R, 64 << 10, 160, 64 << 10, 8192, 0, (1 << R) - 1, None, 0, ctypes.byref(n))
        cuts_us = per_call(lambda: lib.nimbleDebugScheduleDevice(*args))
        merge_us = per_call(lambda: lib.nimbleDebugSchedule(*args), k=10)
        print(f"R={R} per_rank={per >> 20} MiB rank={rank}: {n.value} items; plan {plan_us:.1f} us; "
              f"schedule (cuts) {cuts_us:.1f} us; + host merge {merge_us:.0f} us")
    lib.nimblePlanDestroy(h)
