"""Host cost of building one rank's work-item schedule for a new matrix (nimbleDebugSchedule; development aid)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import planner as P, _lib
lib=_lib.lib()
for R, per in ((8, 256<<20), (8, 16<<20), (4, 256<<20)):
    topo = P.build_canonical(1, R, 0, 900e9, 0, P.NVSWITCH)
    m = P.gen_skewed_a2av(R, per, 0.7, 0)
    off = [0 if i // R == i % R else v for i, v in enumerate(m)]
    cfg = P.PlannerConfig().to_c()
    h = ctypes.c_void_p()
    _lib.call("nimblePlanCreate", topo.handle, R, R, _lib.u64_array(off), ctypes.byref(cfg), ctypes.byref(h))
    n = ctypes.c_int()
    for rank in (0, 1):
        t0=time.perf_counter(); k=20
        for _ in range(k):
            lib.nimbleDebugSchedule(h, rank, R, 64<<10, 160, 64<<10, 8192, 0, (1<<R)-1, None, 0, ctypes.byref(n))
        dt=(time.perf_counter()-t0)/k
        print(f"R={R} per_rank={per>>20}MiB rank={rank}: {n.value} items, build_schedule {dt*1e6:.0f} us")
    lib.nimblePlanDestroy(h)
