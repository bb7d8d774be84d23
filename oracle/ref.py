"""TEST INFRASTRUCTURE ONLY: ctypes access to the compiled reference.

`oracle/_ref/libnimble_ref.so` is the UNMODIFIED reference library
(/root/reference/proj/src/*.cpp) plus the JSON shim `oracle/ref_capi.cpp`,
built by `make -C oracle ref`.  Only tests/, __graft_entry__ and bench.py's
reference / cpu_baseline legs may import this module.
"""
from __future__ import annotations

import ctypes
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libnimble_ref.so")
CPU_SO = os.path.join(HERE, "_build", "liboracle_cpu.so")

_ref = None
_cpu = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _ref
    if _ref is None:
        _ref = ctypes.CDLL(REF_SO)
        _ref.nref_call.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t,
                                   ctypes.POINTER(ctypes.c_size_t)]
        _ref.nref_call.restype = ctypes.c_int
        _ref.nref_time_plan.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
        _ref.nref_time_plan.restype = ctypes.c_double
        _ref.nref_plan_flows.argtypes = [ctypes.c_char_p] + [ctypes.c_void_p] * 4 + [ctypes.c_int]
        _ref.nref_plan_flows.restype = ctypes.c_int
    return _ref


def cpu_lib():
    global _cpu
    if _cpu is None:
        _cpu = ctypes.CDLL(CPU_SO)
        _cpu.orc_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        _cpu.orc_check.argtypes = _cpu.orc_fill.argtypes
        _cpu.orc_check.restype = ctypes.c_uint64
        _cpu.orc_alltoallv.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p]
        _cpu.orc_exchange_flows.argtypes = ([ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_int] +
                                            [ctypes.c_void_p] * 5 +
                                            [ctypes.c_uint64, ctypes.c_int])
        _cpu.orc_exchange_flows.restype = ctypes.c_double
    return _cpu


def call(req: dict) -> dict:
    """Run one reference operation (see oracle/ref_capi.cpp for the ops)."""
    payload = json.dumps(req).encode()
    cap = 1 << 16
    need = ctypes.c_size_t(0)
    while True:
        buf = ctypes.create_string_buffer(cap)
        rc = lib().nref_call(payload, buf, cap, ctypes.byref(need))
        if rc == 2:
            cap = need.value
            continue
        doc = json.loads(buf.value.decode())
        if rc != 0:
            raise RuntimeError(doc.get("error", "reference call failed"))
        return doc


def time_plan(req: dict, warmup: int = 5, runs: int = 100) -> float:
    return lib().nref_time_plan(json.dumps(req).encode(), warmup, runs)


def plan_flows(req: dict, cap: int = 4096):
    """(src, dst, via, bytes) arrays of the reference plan for `req`."""
    src = (ctypes.c_int * cap)()
    dst = (ctypes.c_int * cap)()
    via = (ctypes.c_int * cap)()
    byt = (ctypes.c_double * cap)()
    n = lib().nref_plan_flows(json.dumps(req).encode(), src, dst, via, byt, cap)
    if n < 0:
        raise RuntimeError("reference plan failed")
    return list(src[:n]), list(dst[:n]), list(via[:n]), list(byt[:n])
