"""ctypes binding of libnimble_b200.so (the C ABI declared in include/nimble.h).

The library is built in-tree by `python __graft_entry__.py build` (or `make -C
paper_2604_00317_b200/csrc`).  There is no fallback: if the library is missing
every entry point raises, loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NIMBLE_B200_LIB", os.path.join(HERE, "libnimble_b200.so"))

c_int, c_double, c_u64, c_size, c_void_p, c_char_p = (ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                                     ctypes.c_size_t, ctypes.c_void_p, ctypes.c_char_p)
P = ctypes.POINTER


class NimbleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"nimble error {code}: {msg}")
        self.code = code


class PlannerConfig(ctypes.Structure):  # nimblePlannerConfig
    _fields_ = [("lambda_", c_double), ("epsilon", c_u64), ("pi", c_double),
                ("small_message_cutoff", c_u64), ("saturation_intra", c_u64),
                ("saturation_inter", c_u64), ("max_pair_visits", c_u64),
                ("normalize_by_capacity", c_int)]


class PlanStats(ctypes.Structure):  # nimblePlanStats
    _fields_ = [("pair_visits", c_u64), ("placements", c_u64), ("fallback_pairs", c_u64),
                ("residual_flows", c_u64), ("refine_moves", c_u64), ("wall_seconds", c_double)]


class CommConfig(ctypes.Structure):  # nimbleCommConfig
    _fields_ = [("fabric", c_int), ("gpus_per_node", c_int), ("nvlink_bytes_per_s", c_double),
                ("planner", PlannerConfig), ("pipe_chunk", c_u64), ("p2p_buffer", c_u64),
                ("channels_per_peer", c_int), ("ctas", c_int), ("direct_chunk", c_u64), ("pull", c_int),
                ("push_chunk", c_u64), ("ll_max", c_u64)]


class UniqueId(ctypes.Structure):  # nimbleUniqueId
    _fields_ = [("internal", ctypes.c_char * 128)]


class Item(ctypes.Structure):  # nimbleItem (mirrors the engine's 32-byte work item)
    _fields_ = [("src", c_u64), ("dst", c_u64), ("bytes", ctypes.c_uint32), ("kind", ctypes.c_uint8),
                ("peer", ctypes.c_uint8), ("aux", ctypes.c_uint16), ("seq", ctypes.c_uint32),
                ("pad", ctypes.c_uint32)]


class BenchResult(ctypes.Structure):  # nimbleBenchResult
    _fields_ = [("seconds_median", c_double), ("seconds_min", c_double), ("gbps_effective", c_double),
                ("bound_seconds", c_double), ("plan_seconds", c_double), ("total_bytes", c_u64),
                ("mismatches", c_u64), ("relay_flows", c_int)]


class CommStats(ctypes.Structure):  # nimbleCommStats
    _fields_ = [("bytes", (c_u64 * 32) * 8), ("items", (c_u64 * 32) * 8), ("slot_max_occupancy", c_u64),
                ("slot_double_claims", c_u64), ("slot_claims", c_u64), ("pad", c_u64),
                ("host_calls", c_u64), ("host_ns", c_u64), ("host_ns_max", c_u64), ("plans_built", c_u64),
                ("plan_ns", c_u64), ("schedules_built", c_u64), ("schedule_ns", c_u64), ("host_pad", c_u64)]


# name -> argtypes (restype is always nimbleResult_t unless listed in _RESTYPES)
SIGNATURES = {
    "nimbleGetErrorString": [c_int],
    "nimbleGetLastError": [],
    "nimbleGetVersion": [P(c_int)],
    "nimbleTopologyCreate": [c_int, c_int, c_int, c_double, c_double, c_int, P(c_void_p)],
    "nimbleTopologyLoad": [c_char_p, P(c_void_p)],
    "nimbleTopologySave": [c_void_p, c_char_p, c_size, P(c_size)],
    "nimbleTopologyDestroy": [c_void_p],
    "nimbleTopologyLinkCount": [c_void_p, P(c_int)],
    "nimbleTopologyLink": [c_void_p, c_int, P(c_int), P(c_double), c_char_p, c_size],
    "nimbleTopologySetCapacity": [c_void_p, c_int, c_double],
    "nimbleTopologyLinkId": [c_void_p, c_int, c_int, c_int, c_int, P(c_int)],
    "nimbleGenP2P": [c_int, c_int, c_int, c_u64, P(c_u64)],
    "nimbleGenSkewed": [c_int, c_u64, c_double, c_int, c_int, P(c_u64)],
    "nimbleGenStencil1D": [c_int, c_u64, P(c_u64)],
    "nimbleGenAggregator": [c_int, P(c_int), c_int, c_u64, P(c_u64)],
    "nimbleGenIrregular": [c_int, c_u64, c_double, c_u64, P(c_u64)],
    "nimbleMatrixToText": [c_int, P(c_u64), c_char_p, c_size, P(c_size)],
    "nimbleMatrixFromText": [c_char_p, P(c_u64), c_size, P(c_int)],
    "nimblePlannerConfigDefault": [P(PlannerConfig)],
    "nimblePlanCreate": [c_void_p, c_int, c_int, P(c_u64), P(PlannerConfig), P(c_void_p)],
    "nimblePlanDirect": [c_void_p, c_int, c_int, P(c_u64), P(c_void_p)],
    "nimbleEnumeratePaths": [c_void_p, c_int, c_int, c_int, c_int, P(c_void_p)],
    "nimblePlanDestroy": [c_void_p],
    "nimblePlanNumPairs": [c_void_p, P(c_int)],
    "nimblePlanPair": [c_void_p, c_int, P(c_int), P(c_int), P(c_u64), P(c_int), P(c_int)],
    "nimblePlanCandidate": [c_void_p, c_int, c_int, P(c_int), P(c_int), P(c_int), P(c_int),
                            P(c_int), c_int, P(c_int)],
    "nimblePlanFlow": [c_void_p, c_int, c_int, P(c_int), P(c_double)],
    "nimblePlanGetStats": [c_void_p, P(PlanStats)],
    "nimblePlanLinkLoads": [c_void_p, P(c_double), c_int],
    "nimblePlanMaxNormalizedLoad": [c_void_p, P(c_double)],
    "nimblePlanToJson": [c_void_p, c_char_p, c_size, P(c_size)],
    "nimblePlanFromJson": [c_void_p, c_int, c_int, c_char_p, P(c_void_p)],
    "nimbleCommConfigDefault": [P(CommConfig)],
    "nimbleGetUniqueId": [P(UniqueId)],
    "nimbleCommInitRank": [P(c_void_p), c_int, UniqueId, c_int],
    "nimbleCommInitAll": [P(c_void_p), c_int, P(c_int)],
    "nimbleCommDestroy": [c_void_p],
    "nimbleCommCount": [c_void_p, P(c_int)],
    "nimbleCommUserRank": [c_void_p, P(c_int)],
    "nimbleCommCuDevice": [c_void_p, P(c_int)],
    "nimbleCommGetAsyncError": [c_void_p, P(c_int)],
    "nimbleCommSetConfig": [c_void_p, P(CommConfig)],
    "nimbleCommGetConfig": [c_void_p, P(CommConfig)],
    "nimbleCommRegister": [c_void_p, c_void_p, c_size, P(c_void_p)],
    "nimbleCommDeregister": [c_void_p, c_void_p],
    "nimbleMemAlloc": [P(c_void_p), c_size],
    "nimbleMemFree": [c_void_p],
    "nimbleGroupStart": [],
    "nimbleGroupEnd": [],
    "nimbleSend": [c_void_p, c_size, c_int, c_int, c_void_p, c_void_p],
    "nimbleRecv": [c_void_p, c_size, c_int, c_int, c_void_p, c_void_p],
    "nimbleAlltoAll": [c_void_p, c_void_p, c_size, c_int, c_void_p, c_void_p],
    "nimbleAlltoAllv": [c_void_p, P(c_size), P(c_size), c_void_p, P(c_size), P(c_size), c_int,
                        c_void_p, c_void_p],
    "nimbleExchangeLocal": [c_int, P(c_void_p), P(c_void_p), P(c_u64), c_int, c_void_p],
    "nimbleFillPayload": [c_void_p, c_u64, c_u64, c_u64, c_int, c_int, c_void_p],
    "nimbleCheckPayload": [c_void_p, c_u64, c_u64, c_u64, c_int, c_int, c_void_p, c_void_p],
    "nimbleBenchP2P": [c_void_p, c_u64, c_int, c_int, c_int, c_int, P(BenchResult)],
    "nimbleBenchSkewed": [c_void_p, c_u64, c_double, c_int, c_int, c_int, P(BenchResult)],
    "nimbleBenchMatrix": [c_void_p, P(c_u64), c_int, c_int, P(BenchResult)],
    "nimbleBootstrapAllgather": [P(UniqueId), c_int, c_int, c_void_p, c_size, c_void_p],
    "nimbleBootstrapShmAllgather": [P(UniqueId), c_int, c_int, c_void_p, c_size, c_void_p, c_int],
    "nimbleCommDebugTrace": [c_void_p, P(c_u64), c_int],
    "nimbleCommGetStats": [c_void_p, P(CommStats), c_int],
    "nimbleDebugSchedule": [c_void_p, c_int, c_int, c_u64, ctypes.c_uint32, c_u64, c_u64, c_u64, c_u64, c_void_p, c_int,
                            P(c_int)],
    "nimbleDebugScheduleDevice": [c_void_p, c_int, c_int, c_u64, ctypes.c_uint32, c_u64, c_u64, c_u64, c_u64, c_void_p,
                                  c_int, P(c_int)],
}
_RESTYPES = {"nimbleGetErrorString": c_char_p, "nimbleGetLastError": c_char_p}

_lib = None


def lib():
    """Load the in-tree library once; raise if it is absent (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build`")
        handle = ctypes.CDLL(LIB_PATH)
        missing = [n for n in SIGNATURES if not hasattr(handle, n)]
        if missing and not os.environ.get("NIMBLE_B200_PARTIAL"):
            raise ImportError(f"{LIB_PATH} lacks exported symbols: {missing}")
        for name, args in SIGNATURES.items():
            if name in missing:
                continue
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, c_int)
        _lib = handle
    return _lib


def check(code: int):
    if code != 0:
        raise NimbleError(code, lib().nimbleGetLastError().decode(errors="replace"))


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def u64_array(values):
    arr = (c_u64 * len(values))()
    for i, v in enumerate(values):
        arr[i] = int(v)
    return arr
