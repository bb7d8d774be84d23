"""Python face of the NCCL-shaped communicator (include/nimble.h group 2/3).

Thin ctypes wrappers: every data-path call goes straight to
libnimble_b200.so, which launches the sm_100a forwarding engine.  Tensors are
only used for their device pointers and streams (PyTorch is plumbing here).
"""
from __future__ import annotations

import contextlib
import ctypes

from . import _lib
from ._lib import c_double, c_int, c_size, c_u64, c_void_p

UINT8 = 1  # nimbleUint8


def _load_fast():
    """The CPython fast call into nimbleAlltoAllv (csrc/pyfast.cpp), bound to the
    function of the library _lib loaded; None if the module was not built."""
    try:
        from . import _fast
    except ImportError:
        return None
    _fast.init(ctypes.cast(_lib.lib().nimbleAlltoAllv, c_void_p).value)
    return _fast


_FAST = _load_fast()


def _ptr(t) -> int:
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


def _current_stream() -> int:
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # no Stream object per call
    if raw is not None:
        return raw(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def _stream_handle(stream) -> int:
    if stream is None:
        return _current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


_SIZE_ARRAYS: dict = {}


def _sizes(values):
    n = len(values)
    t = _SIZE_ARRAYS.get(n)
    if t is None:
        t = _SIZE_ARRAYS[n] = c_size * n
    return t(*values)


def unique_id() -> bytes:
    uid = _lib.UniqueId()
    _lib.call("nimbleGetUniqueId", ctypes.byref(uid))
    return ctypes.string_at(ctypes.addressof(uid), ctypes.sizeof(uid))


def comm_config_default() -> _lib.CommConfig:
    cfg = _lib.CommConfig()
    _lib.call("nimbleCommConfigDefault", ctypes.byref(cfg))
    return cfg


class Comm:
    """One rank of a communicator (nimbleCommInitRank / nimbleCommInitAll)."""

    def __init__(self, handle):
        self._h = c_void_p(handle) if not isinstance(handle, c_void_p) else handle
        self._hv = self._h.value  # plain int for the fast call
        n, r, d = c_int(), c_int(), c_int()
        _lib.call("nimbleCommCount", self._h, ctypes.byref(n))
        _lib.call("nimbleCommUserRank", self._h, ctypes.byref(r))
        _lib.call("nimbleCommCuDevice", self._h, ctypes.byref(d))
        self.nranks, self.rank, self.device = n.value, r.value, d.value

    @classmethod
    def init_rank(cls, nranks: int, uid: bytes, rank: int) -> "Comm":
        u = _lib.UniqueId()
        ctypes.memmove(ctypes.addressof(u), uid, min(len(uid), ctypes.sizeof(u)))
        h = c_void_p()
        _lib.call("nimbleCommInitRank", ctypes.byref(h), nranks, u, rank)
        return cls(h)

    @classmethod
    def init_all(cls, devices) -> list:
        n = len(devices)
        arr = (c_void_p * n)()
        devs = (c_int * n)(*devices)
        _lib.call("nimbleCommInitAll", arr, n, devs)
        return [cls(c_void_p(arr[i])) for i in range(n)]

    def destroy(self):
        if self._h:
            _lib.call("nimbleCommDestroy", self._h)
            self._h = None
            self._hv = 0

    @property
    def handle(self):
        return self._h

    # -- configuration
    def config(self) -> _lib.CommConfig:
        cfg = _lib.CommConfig()
        _lib.call("nimbleCommGetConfig", self._h, ctypes.byref(cfg))
        return cfg

    def set_config(self, cfg: _lib.CommConfig | None = None, **fields):
        cfg = cfg or self.config()
        for k, v in fields.items():
            if k == "fabric" and isinstance(v, str):
                v = 0 if v == "alltoall" else 1
            setattr(cfg, k, v)
        _lib.call("nimbleCommSetConfig", self._h, ctypes.byref(cfg))

    def async_error(self) -> int:
        e = c_int()
        _lib.call("nimbleCommGetAsyncError", self._h, ctypes.byref(e))
        return e.value

    def check_async(self):
        e = self.async_error()
        if e:
            raise _lib.NimbleError(e, _lib.lib().nimbleGetLastError().decode())

    def debug_trace(self, per_cta=False):
        """Device timeline (ns) of the last launch; needs NIMBLE_TRACE=1.
        per_cta: also the per-CTA words (include/nimble.h), as a second list
        of [first, queue_empty, loops_done, fence_done, remote_bytes,
        other_bytes] rows for the CTAs that ran."""
        n = 16 + 160 * 6 if per_cta else 16
        out = (c_u64 * n)()
        _lib.call("nimbleCommDebugTrace", self._h, out, n)
        v = list(out)
        if not per_cta:
            return v
        rows = [v[16 + 6 * i:22 + 6 * i] for i in range(160)]
        return v[:16], [r for r in rows if r[2]]

    STAT_KINDS = ("local", "push", "stage", "forward", "pull", "ll_send", "ll_recv", "drain")

    def stats(self, reset=False) -> dict:
        """Engine counters since creation / the last reset (needs NIMBLE_STATS=1
        when the comm was created): bytes and items per (kind, peer) and the
        staging rings' slot-occupancy check (include/nimble.h)."""
        st = _lib.CommStats()
        _lib.call("nimbleCommGetStats", self._h, ctypes.byref(st), 1 if reset else 0)
        out = {"slot_max_occupancy": st.slot_max_occupancy, "slot_double_claims": st.slot_double_claims,
               "slot_claims": st.slot_claims, "host_calls": st.host_calls, "host_ns": st.host_ns,
               "host_ns_max": st.host_ns_max, "plans_built": st.plans_built, "plan_ns": st.plan_ns,
               "schedules_built": st.schedules_built, "schedule_ns": st.schedule_ns}
        for k, name in enumerate(self.STAT_KINDS):
            out[name] = [int(st.bytes[k][p]) for p in range(self.nranks)]
            out[name + "_items"] = [int(st.items[k][p]) for p in range(self.nranks)]
        return out

    # -- registration
    def register(self, tensor, nbytes=None):
        h = c_void_p()
        n = nbytes if nbytes is not None else tensor.numel() * tensor.element_size()
        _lib.call("nimbleCommRegister", self._h, c_void_p(_ptr(tensor)), n, ctypes.byref(h))
        return h

    def deregister(self, handle):
        _lib.call("nimbleCommDeregister", self._h, handle)

    # -- data path (counts / displacements in bytes: uint8 datatype)
    def alltoallv(self, send, sendcounts, sdispls, recv, recvcounts, rdispls, stream=None, datatype=UINT8):
        n = self.nranks
        if len(sendcounts) != n or len(sdispls) != n or len(recvcounts) != n or len(rdispls) != n:
            raise ValueError(f"alltoallv: counts and displacements need exactly {n} entries (one per rank)")
        if _FAST is not None:  # same C entry point, without ctypes' per-call conversions
            rc = _FAST.alltoallv(self._hv, _ptr(send), sendcounts, sdispls, _ptr(recv), recvcounts, rdispls,
                                 datatype, _stream_handle(stream))
        else:
            rc = _lib.lib().nimbleAlltoAllv(_ptr(send), _sizes(sendcounts), _sizes(sdispls), _ptr(recv),
                                            _sizes(recvcounts), _sizes(rdispls), datatype, self._h,
                                            _stream_handle(stream))
        _lib.check(rc)

    def alltoall(self, send, recv, count, stream=None, datatype=UINT8):
        _lib.call("nimbleAlltoAll", c_void_p(_ptr(send)), c_void_p(_ptr(recv)), count, datatype, self._h,
                  c_void_p(_stream_handle(stream)))

    def send(self, buf, nbytes, peer, stream=None):
        _lib.call("nimbleSend", c_void_p(_ptr(buf)), nbytes, UINT8, peer, self._h,
                  c_void_p(_stream_handle(stream)))

    def recv(self, buf, nbytes, peer, stream=None):
        _lib.call("nimbleRecv", c_void_p(_ptr(buf)), nbytes, UINT8, peer, self._h,
                  c_void_p(_stream_handle(stream)))

    # -- bench entry points (--p2p / --skewed)
    def _bench(self, name, *args):
        res = _lib.BenchResult()
        _lib.call(name, self._h, *args, ctypes.byref(res))
        return {k: getattr(res, k) for k, _ in _lib.BenchResult._fields_}

    def bench_p2p(self, nbytes, src=0, dst=1, warmup=3, iters=10):
        return self._bench("nimbleBenchP2P", nbytes, src, dst, warmup, iters)

    def bench_skewed(self, per_rank, ratio, hot=0, warmup=3, iters=10):
        return self._bench("nimbleBenchSkewed", per_rank, float(ratio), hot, warmup, iters)

    def bench_matrix(self, matrix, warmup=3, iters=10):
        return self._bench("nimbleBenchMatrix", _lib.u64_array(matrix), warmup, iters)


@contextlib.contextmanager
def group():
    """nimbleGroupStart / nimbleGroupEnd."""
    _lib.call("nimbleGroupStart")
    try:
        yield
    finally:
        _lib.call("nimbleGroupEnd")


def exchange_local(sends, recvs, matrix, ctas=0, stream=None):
    """nimbleExchangeLocal: the R-rank exchange emulated on one GPU."""
    R = len(sends)
    s = (c_void_p * R)(*[_ptr(t) for t in sends])
    r = (c_void_p * R)(*[_ptr(t) for t in recvs])
    _lib.call("nimbleExchangeLocal", R, s, r, _lib.u64_array(matrix), ctas, c_void_p(_stream_handle(stream)))


def fill_payload(buf, first, nbytes, seed, src, dst, stream=None):
    _lib.call("nimbleFillPayload", c_void_p(_ptr(buf)), first, nbytes, seed, src, dst,
              c_void_p(_stream_handle(stream)))


def check_payload(buf, first, nbytes, seed, src, dst, counter, stream=None):
    """Adds the number of mismatching bytes into `counter` (a 1-element int64 CUDA tensor)."""
    _lib.call("nimbleCheckPayload", c_void_p(_ptr(buf)), first, nbytes, seed, src, dst,
              c_void_p(_ptr(counter)), c_void_p(_stream_handle(stream)))


def packed_displs(matrix, R, me):
    """Packed MPI layout for rank `me`: (sendcounts, sdispls, recvcounts, rdispls)."""
    sc = [matrix[me * R + d] for d in range(R)]
    rc = [matrix[s * R + me] for s in range(R)]
    sd, rd, a, b = [], [], 0, 0
    for d in range(R):
        sd.append(a)
        a += sc[d]
    for s in range(R):
        rd.append(b)
        b += rc[s]
    return sc, sd, rc, rd
