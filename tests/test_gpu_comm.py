"""Parity of the NVLink data path, bit-exact against the payload function
and the host oracle (oracle/cpu_exchange.c orc_alltoallv).

Two ways to run R ranks:
  - "proc": one process per GPU (gpurun --gpus 2|4), the production layout;
  - "thread": R ranks co-resident on ONE GPU -- one process, one thread and
    one stream per rank, nimbleCommInitRank over the same bootstrap.  The comm
    sizes every rank's engine grid to (SMs - R) / R CTAs so all R grids are
    resident at once; peers' ctrl / staging / registered windows are plain
    pointers into the same HBM.  Every part of the cross-rank protocol runs
    (posts, ready / consumed ring flags, pushes, TMA pulls, LL slots, relay
    rings, completion counters) -- only the wire is HBM instead of NVLink.
    This is how a 1-GPU box runs the 2/4/8-rank protocol tests.
"""
import os
import socket
import threading
import traceback

import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu]

MiB = 1 << 20
_CALL_TIMEOUT_S = 600


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


# ---------------------------------------------------------------- rank context

_CTX = threading.local()  # .mode ("proc" | "thread"), .barrier (thread mode)


def _sync():
    """Wait for this rank's work.  In thread mode only the rank's own stream:
    a device-wide sync would also wait for peer grids that may be waiting for
    this rank's next launch."""
    if getattr(_CTX, "mode", "proc") == "thread":
        torch.cuda.current_stream().synchronize()
    else:
        torch.cuda.synchronize()


def _barrier():
    if getattr(_CTX, "mode", "proc") == "thread":
        _CTX.barrier.wait(timeout=_CALL_TIMEOUT_S)
    else:
        import torch.distributed as dist
        dist.barrier()


def _capture(fn):
    """CUDA-graph capture of fn() on a private stream, thread-local capture mode
    (other ranks' threads keep running), no device-wide sync."""
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin(capture_error_mode="thread_local")
        try:
            fn()
        finally:
            g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    return g


def _worker(fn):
    """A worker of this module by name, or "module:function" (debug tools)."""
    if ":" in fn:
        import importlib
        mod, name = fn.split(":")
        return getattr(importlib.import_module(mod), name)
    return globals()[fn]


# ---------------------------------------------------------------- process mode

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        rank, res = q.get(timeout=_CALL_TIMEOUT_S)
        out[rank] = res
    for p in procs:
        p.join(timeout=120)
    for r, res in out.items():
        if isinstance(res, str) and res.startswith("ERROR"):
            pytest.fail(f"rank {r}: {res}")
    return out


def _entry(fn, rank, world, port, q, args):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NIMBLE_TIMEOUT_MS="15000",
                          NIMBLE_STATS="1")
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        _CTX.mode = "proc"
        from paper_2604_00317_b200 import comm as C
        uid = [C.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, 0)
        comm = C.Comm.init_rank(world, uid[0], rank)
        res = _worker(fn)(comm, rank, world, *args)
        dist.barrier()
        comm.destroy()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:
        q.put((rank, "ERROR " + traceback.format_exc()))


# ---------------------------------------------------------------- thread mode (co-resident on GPU 0)

def _thread_server(R, conn):
    """Long-lived child process: runs worker calls as R threads on GPU 0."""
    # one hardware queue per stream: R ranks' streams must not alias onto one
    # queue (a spinning grid would block the peer grid queued behind it)
    # (a rank that failed leaves the others in a host collective: fail fast)
    os.environ.update(NIMBLE_TIMEOUT_MS="15000", NIMBLE_STATS="1", CUDA_DEVICE_MAX_CONNECTIONS="32",
                      NIMBLE_BOOTSTRAP_TIMEOUT_MS="60000", NIMBLE_TRACE="1")
    torch.cuda.set_device(0)
    from paper_2604_00317_b200 import comm as C
    while True:
        msg = conn.recv()
        if msg is None:
            break
        fn, args = msg
        uid = C.unique_id()
        barrier = threading.Barrier(R)
        out = [None] * R

        def run(rank):
            try:
                torch.cuda.set_device(0)
                _CTX.mode, _CTX.barrier = "thread", barrier
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    _warm_allocator(R)
                    comm = None
                    comm = C.Comm.init_rank(R, uid, rank)
                    out[rank] = _worker(fn)(comm, rank, R, *args)
                    s.synchronize()
                    barrier.wait(timeout=_CALL_TIMEOUT_S)
                    comm.destroy()
            except Exception as e:
                if isinstance(e, threading.BrokenBarrierError):
                    out[rank] = "ERROR (another rank failed first)"
                else:
                    err = ""
                    try:
                        err = f" [async error {comm.async_error()}]"
                        t = comm.debug_trace()  # last launch: kernel start / done (globaltimer, one GPU)
                        err += f" [last launch start {t[0] % 10**10} waited {t[6] % 10**10} ns]"
                    except Exception:
                        pass
                    out[rank] = "ERROR" + err + " " + traceback.format_exc()
                barrier.abort()

        threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(R)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        conn.send(out)


_SERVERS = {}


def _warm_allocator(R):
    """Fill this thread's stream with cached device memory before any
    exchange (16 GiB per server, split over its ranks).  A cudaMalloc
    issued while peer ranks' engines spin on this
    rank's flags can keep this rank's next kernel from starting (device
    memory allocation is one of CUDA's implicit synchronization points
    between streams): the workers' tensors must come from the cache."""
    big = torch.empty((16 << 30) // R, dtype=torch.uint8, device="cuda")
    small = [torch.empty(256 << 10, dtype=torch.uint8, device="cuda") for _ in range(64)]
    del big, small
    torch.cuda.current_stream().synchronize()


def _server(R):
    import multiprocessing as mp
    for other in [r for r in _SERVERS if r != R]:  # one server (and its cached HBM) at a time
        _stop(other)
    srv = _SERVERS.get(R)
    if srv is None or not srv[0].is_alive():
        ctx = mp.get_context("spawn")
        parent, child = ctx.Pipe()
        p = ctx.Process(target=_thread_server, args=(R, child), daemon=True)
        # Eager module loading in the server (set before its CUDA init, which
        # importing this module already does): CUDA loads a kernel's module on
        # its first launch, and a module load waits for the device's running
        # kernels -- here peer ranks' engines spinning on this rank's next
        # exchange, so a torch kernel first used between two exchanges stalled
        # them until their timeout (tools/first_use_probe.py).
        prev = os.environ.get("CUDA_MODULE_LOADING")
        os.environ["CUDA_MODULE_LOADING"] = "EAGER"
        try:
            p.start()
        finally:
            if prev is None:
                os.environ.pop("CUDA_MODULE_LOADING")
            else:
                os.environ["CUDA_MODULE_LOADING"] = prev
        srv = _SERVERS[R] = (p, parent)
    return srv


def _kill(R):
    p, conn = _SERVERS.pop(R)
    p.kill()
    p.join(timeout=30)


def _stop(R):
    p, conn = _SERVERS.pop(R)
    try:
        conn.send(None)
        p.join(timeout=30)
    except Exception:
        pass
    if p.is_alive():
        p.kill()
        p.join(timeout=30)


@pytest.fixture(scope="module", autouse=True)
def _stop_servers():
    yield
    for R in list(_SERVERS):
        _stop(R)


def _threads(fn, R, *args):
    p, conn = _server(R)
    conn.send((fn, args))
    if not conn.poll(_CALL_TIMEOUT_S):
        _kill(R)
        pytest.fail(f"{fn} at R={R} (co-resident): no result within {_CALL_TIMEOUT_S} s")
    try:
        out = conn.recv()
    except EOFError:
        _kill(R)
        pytest.fail(f"{fn} at R={R} (co-resident): server died")
    errors = [(r, v) for r, v in enumerate(out) if isinstance(v, str) and v.startswith("ERROR")]
    if errors:
        _kill(R)  # ranks may be stuck in a collective: start over
        pytest.fail("\n".join(f"rank {r}: {v}" for r, v in errors))
    return dict(enumerate(out))


def _run(layout, fn, *args):
    mode, R = layout
    return _threads(fn, R, *args) if mode == "thread" else _spawn(fn, R, *args)


def _layouts(*thread_ranks, proc=True, proc_min=2, proc_max=4):
    """pytest params: co-resident thread layouts (any GPU box) + the one-process-
    per-GPU layout on a multi-GPU box."""
    out = [pytest.param(("thread", r), id=f"thread{r}") for r in thread_ranks]
    if proc:
        n = min(_ngpus(), proc_max)
        out.append(pytest.param(("proc", max(n, proc_min)), id="proc",
                                marks=[pytest.mark.multigpu,
                                       pytest.mark.skipif(n < proc_min, reason=f"needs >= {proc_min} GPUs")]))
    return out


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _host_check(rank, R, m, seed, recv):
    """Rank `rank`'s receive buffer, copied to the host, against the host
    oracle's orc_alltoallv of the same matrix over the payload bytes."""
    import ctypes
    import numpy as np
    from oracle import ref
    lib = ref.cpu_lib()
    sends = []
    for s in range(R):
        row = [m[s * R + d] for d in range(R)]
        buf = np.zeros(max(sum(row), 1), dtype=np.uint8)
        off = 0
        for d in range(R):
            lib.orc_fill(buf[off:].ctypes.data_as(ctypes.c_void_p), 0, row[d], seed, s, d)
            off += row[d]
        sends.append(buf)
    want = [np.zeros(max(sum(m[s * R + d] for s in range(R)), 1), dtype=np.uint8) for d in range(R)]
    mat = (ctypes.c_uint64 * (R * R))(*m)
    lib.orc_alltoallv(R, mat, (ctypes.c_void_p * R)(*[b.ctypes.data for b in sends]),
                      (ctypes.c_void_p * R)(*[w.ctypes.data for w in want]))
    n = sum(m[s * R + rank] for s in range(R))
    _sync()
    got = recv[:n].cpu().numpy()
    return int((got != want[rank][:n]).sum())


def _slots(comm):
    cfg = comm.config()
    return cfg.channels_per_peer * (cfg.p2p_buffer // cfg.pipe_chunk)


def _rings_bounded(comm):
    """Device-side bounded-buffer check of every staging ring this rank fed
    since the comm's counters were last reset (reference
    tests/acceptance.cpp:270-288: occupancy <= S; and no slot claimed while
    its previous chunk was undrained)."""
    st = comm.stats()
    return st["slot_double_claims"] == 0 and st["slot_max_occupancy"] <= _slots(comm)


def _exchange_and_check(comm, rank, R, m, register, seed, register_send=False, host_check=True):
    from paper_2604_00317_b200 import comm as C
    sc, sd, rc, rd = C.packed_displs(m, R, rank)
    send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
    recv = torch.full((max(sum(rc), 16),), 0xEE, dtype=torch.uint8, device="cuda")
    for d in range(R):
        C.fill_payload(send[sd[d]:], 0, sc[d], seed, rank, d)
    h = comm.register(recv) if register else None
    hs = comm.register(send) if register_send else None
    comm.alltoallv(send, sc, sd, recv, rc, rd)
    _sync()
    comm.check_async()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s in range(R):
        C.check_payload(recv[rd[s]:], 0, rc[s], seed, s, rank, bad)
    # bytes past the packed segments are untouched
    tail_ok = bool((recv[sum(rc):] == 0xEE).all()) if recv.numel() > sum(rc) else True
    _sync()
    # rank 0's buffer on the host against the oracle's all-to-allv (bounded size)
    if host_check and rank == 0 and sum(m) <= 512 * MiB:
        tail_ok = tail_ok and _host_check(rank, R, m, seed, recv) == 0
    tail_ok = tail_ok and _rings_bounded(comm)
    if h is not None:
        comm.deregister(h)
    if hs is not None:
        comm.deregister(hs)
    return int(bad.item()), tail_ok


def w_skewed(comm, rank, R, per_rank, ratio, register):
    from paper_2604_00317_b200 import planner as P
    m = P.gen_skewed_a2av(R, per_rank, ratio, 0)
    return _exchange_and_check(comm, rank, R, m, register, 11)


def _ragged_matrix(R, seed):
    """A seeded ragged matrix (identical on every rank): zero pairs, 1-byte
    pairs, pairs around the LL piece (8 KiB) and the LL limit (1 MiB), and
    multi-MiB pairs, with the self segment too."""
    import random
    rng = random.Random(seed)
    sizes = [0, 0, 1, 7, 8191, 8193, (1 << 20) - 1, (1 << 20), (1 << 20) + 1, 3 * MiB + 5, 9 * MiB + 333]
    return [rng.choice(sizes) for _ in range(R * R)]


def w_ragged_fuzz(comm, rank, R, seeds):
    """Ragged matrices at odd rank counts, each under three registration
    layouts (receive windows registered everywhere / nowhere / on odd ranks
    only -- staged and zero-copy receivers in one exchange), send windows
    registered so receivers may pull: bit-exact on the device, rank 0 on the
    host against orc_alltoallv, rings bounded."""
    from paper_2604_00317_b200 import comm as C
    out = []
    for seed in seeds:
        m = _ragged_matrix(R, seed)
        for layout in ("all", "none", "odd"):
            sc, sd, rc, rd = C.packed_displs(m, R, rank)
            send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
            recv = torch.full((max(sum(rc), 16),), 0xEE, dtype=torch.uint8, device="cuda")
            scratch = torch.empty(4096, dtype=torch.uint8, device="cuda")
            for d in range(R):
                C.fill_payload(send[sd[d]:], 0, sc[d], seed, rank, d)
            mine = layout == "all" or (layout == "odd" and rank % 2 == 1)
            # registration is collective (one buffer per rank per call): the
            # ranks that stay staged register a scratch buffer instead
            hr = comm.register(recv if mine else scratch) if layout != "none" else None
            hs = comm.register(send)
            for _ in range(2):  # twice: the second call reuses the cached schedule (and chains)
                comm.alltoallv(send, sc, sd, recv, rc, rd)
            _sync()
            comm.check_async()
            bad = torch.zeros(1, dtype=torch.int64, device="cuda")
            for s_ in range(R):
                C.check_payload(recv[rd[s_]:], 0, rc[s_], seed, s_, rank, bad)
            _sync()
            ok = int(bad.item()) == 0 and _rings_bounded(comm)
            if rank == 0:
                ok = ok and _host_check(rank, R, m, seed, recv) == 0
            out.append(ok)
            if hr is not None:
                comm.deregister(hr)
            comm.deregister(hs)
            _barrier()
    return out


def w_pull_modes(comm, rank, R):
    """Receiver-driven pulls: every (pull mode, send registered, recv registered)
    combination delivers bit-exactly (granted pulls, declined pulls falling back
    to zero-copy or staged pushes)."""
    from paper_2604_00317_b200 import planner as P
    out = []
    for pull in (0, 1, 2):
        comm.set_config(pull=pull)
        for reg_send in (True, False):
            for reg_recv in (True, False):
                for ratio in (0.9, 1.0 / (R - 1)):
                    m = P.gen_skewed_a2av(R, 6 * MiB + 7, ratio, 1 % R)
                    out.append(_exchange_and_check(comm, rank, R, m, reg_recv, 31, reg_send))
    comm.set_config(pull=0)
    return out


def w_irregular(comm, rank, R):
    from paper_2604_00317_b200 import planner as P
    out = []
    for total in (1024, 65536, 4 * MiB + 3, 64 * MiB):
        for register in (True, False):
            out.append(_exchange_and_check(comm, rank, R, P.gen_irregular(R, total, 0.5, 1), register, total))
    return out


def w_repeat_mixed(comm, rank, R):
    """Back-to-back exchanges on one stream, alternating registered / staged
    receive buffers and matrices (epochs, flag tags, schedule cache)."""
    from paper_2604_00317_b200 import planner as P
    res = []
    for it in range(8):
        m = P.gen_skewed_a2av(R, (3 + it) * MiB + it, 0.3 + 0.1 * it, it % R)
        res.append(_exchange_and_check(comm, rank, R, m, it % 2 == 0, 100 + it, it % 4 < 2))
    return res


def w_stress_back_to_back(comm, rank, R):
    """Many exchanges queued back to back without host syncs: alternating
    matrices, buffers, registrations and push/pull modes (epoch-parity posts,
    flag tags, schedule cache), each verified afterwards."""
    import random
    from paper_2604_00317_b200 import comm as C
    from paper_2604_00317_b200 import planner as P
    rng = random.Random(7)  # same sequence on every rank
    pool = []
    for it in range(3):
        m = P.gen_skewed_a2av(R, (1 + 3 * it) * MiB + 11 * it, 0.2 + 0.3 * it, it % R)
        sc, sd, rc, rd = C.packed_displs(m, R, rank)
        send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
        for d in range(R):
            C.fill_payload(send[sd[d]:], 0, sc[d], 50 + it, rank, d)
        recvs = [torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda") for _ in range(2)]
        hs = comm.register(send) if it != 1 else None
        hr = comm.register(recvs[0])
        pool.append((m, sc, sd, rc, rd, send, recvs, hs, hr, 50 + it))
    plan = [(rng.randrange(3), rng.randrange(2), rng.choice([1, 2])) for _ in range(40)]
    for k, (i, j, pull) in enumerate(plan):
        if k % 10 == 0:
            comm.set_config(pull=pull)  # a config change is a (host-synchronizing) collective
        m, sc, sd, rc, rd, send, recvs, hs, hr, seed = pool[i]
        comm.alltoallv(send, sc, sd, recvs[j], rc, rd)
    _sync()
    comm.check_async()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for (m, sc, sd, rc, rd, send, recvs, hs, hr, seed) in pool:
        for j in range(2):
            if any(pi == pool.index((m, sc, sd, rc, rd, send, recvs, hs, hr, seed)) and pj == j for pi, pj, _ in plan):
                for s in range(R):
                    C.check_payload(recvs[j][rd[s]:], 0, rc[s], seed, s, rank, bad)
    _sync()
    for (m, sc, sd, rc, rd, send, recvs, hs, hr, seed) in pool:
        if hs is not None:
            comm.deregister(hs)
        comm.deregister(hr)
    return int(bad.item())


def w_sendrecv_ring(comm, rank, R):
    from paper_2604_00317_b200 import comm as C
    n = 5 * MiB + 17
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    C.fill_payload(x, 0, n, 5, rank, (rank + 1) % R)
    y = torch.zeros(n, dtype=torch.uint8, device="cuda")
    with C.group():
        comm.send(x, n, (rank + 1) % R)
        comm.recv(y, n, (rank - 1) % R)
    _sync()
    comm.check_async()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    C.check_payload(y, 0, n, 5, (rank - 1) % R, rank, bad)
    _sync()
    return int(bad.item())


def w_relay(comm, rank, R, nbytes):
    """Mesh model: the planner routes p2p 0 -> 1 through relays 2..R-1; the
    engine executes the relay hops through the staging rings."""
    from paper_2604_00317_b200 import planner as P
    comm.set_config(fabric="alltoall", gpus_per_node=R)
    m = P.gen_p2p(R, 0, 1, nbytes)
    res = _exchange_and_check(comm, rank, R, m, True, 21)
    b = comm.bench_p2p(nbytes, 0, 1, warmup=1, iters=2)
    comm.set_config(fabric="nvswitch")
    return res, b["relay_flows"], b["mismatches"]


def w_mismatch(comm, rank, R):
    """Receiver expects fewer bytes than the sender sends: async error, no hang."""
    from paper_2604_00317_b200 import comm as C
    n = 1 * MiB
    x = torch.zeros(n, dtype=torch.uint8, device="cuda")
    y = torch.zeros(n, dtype=torch.uint8, device="cuda")
    h = comm.register(y)
    sc = [n if d != rank else 0 for d in range(R)]
    rc = [n - (1 if rank == 1 else 0) if s != rank else 0 for s in range(R)]
    sd, rd = [0] * R, [0] * R
    try:
        comm.alltoallv(x, sc, sd, y, rc, rd)
        _sync()
    except Exception as e:  # host-side detection is acceptable too
        return "raised: " + str(e)[:60]
    return comm.async_error()


def w_moe(comm, rank, R):
    """MoE dispatch/combine over the nimble all-to-allv (upstream caller):
    skewed router, expert fn = scale by (global expert id + 1), router-weighted
    combine, compared with the same computation done locally."""
    from paper_2604_00317_b200.moe import MoEDispatcher
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    T, H, k, E = 777, 96, 2, 4 * R
    x = torch.randn(T, H, device="cuda", generator=g)
    hot = torch.rand(T, k, device="cuda", generator=g) < 0.6
    ids = torch.where(hot, torch.zeros_like(hot, dtype=torch.int64),
                      torch.randint(0, E, (T, k), device="cuda", generator=g))
    w = torch.rand(T, k, device="cuda", generator=g)
    disp = MoEDispatcher(comm, E, H, dtype=torch.float32, max_tokens=1024, topk=k)
    try:
        recv_x, recv_e, h = disp.dispatch(x, ids)
        y = recv_x * (recv_e.to(torch.float32) + rank * disp.experts_per_rank + 1).unsqueeze(1)
        out = disp.combine(y, h, w)
        _sync()
        comm.check_async()
        ref = (x.unsqueeze(1) * (ids.to(torch.float32) + 1).unsqueeze(2) * w.unsqueeze(2)).sum(1)
        ok = torch.allclose(out, ref, rtol=1e-5, atol=1e-5)
        return bool(ok), sum(h.recv_counts)
    finally:
        disp.close()


def w_graph(comm, rank, R):
    """An exchange captured in a CUDA graph and replayed: each replay takes a
    fresh epoch from device memory, so every replay delivers correctly."""
    from paper_2604_00317_b200 import comm as C
    from paper_2604_00317_b200 import planner as P
    m = P.gen_skewed_a2av(R, 8 * MiB + 3, 0.7, 0)
    sc, sd, rc, rd = C.packed_displs(m, R, rank)
    send = torch.empty(sum(sc), dtype=torch.uint8, device="cuda")
    recv = torch.zeros(sum(rc), dtype=torch.uint8, device="cuda")
    hs, hr = comm.register(send), comm.register(recv)
    comm.alltoallv(send, sc, sd, recv, rc, rd)  # warm-up: the schedule is cached before capture
    _sync()
    g = _capture(lambda: comm.alltoallv(send, sc, sd, recv, rc, rd))
    _barrier()  # every rank captured before any rank replays
    bads = []
    for i in range(5):
        for d in range(R):
            C.fill_payload(send[sd[d]:], 0, sc[d], 200 + i, rank, d)
        recv.zero_()
        _sync()
        g.replay()
        _sync()
        bad = torch.zeros(1, dtype=torch.int64, device="cuda")
        for s in range(R):
            C.check_payload(recv[rd[s]:], 0, rc[s], 200 + i, s, rank, bad)
        _sync()
        bads.append(int(bad.item()))
    comm.check_async()
    comm.alltoallv(send, sc, sd, recv, rc, rd)  # eager launches keep working after replays
    _sync()
    # The graph pins its schedule: more distinct exchanges than the schedule
    # cache holds, then a deregistration (which drops every cached schedule),
    # must leave the captured launch's buffers alive.
    extra = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    hx = comm.register(extra)
    for k in range(6):
        mk = P.gen_skewed_a2av(R, MiB + 97 * k, 0.5, 0)
        a, b, c_, d_ = C.packed_displs(mk, R, rank)
        comm.alltoallv(send, a, b, recv, c_, d_)
    _sync()
    comm.deregister(hx)
    _barrier()
    for d in range(R):
        C.fill_payload(send[sd[d]:], 0, sc[d], 300, rank, d)
    recv.zero_()
    _sync()
    g.replay()
    _sync()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s in range(R):
        C.check_payload(recv[rd[s]:], 0, rc[s], 300, s, rank, bad)
    _sync()
    bads.append(int(bad.item()))
    comm.check_async()
    comm.deregister(hs)
    comm.deregister(hr)
    return bads


def w_overtake(comm, rank, R, big, small):
    """Post slots are double-buffered by epoch parity.  A receiver that pulled
    everything it needed from a sender does not wait for that sender, so it
    can run two launches ahead and overwrite the post slot the sender has not
    read yet.  The sender must infer the pull from the newer epoch instead of
    waiting for a post that never comes back.  Here rank 1 is held in launch A
    by a `big` self copy whose items surround its small segment for rank 0.
    Rank 0 pulls that segment, runs launch B (its own self copy only), and
    then launch C, whose post for rank 1 lands in A's slot.  With `small` under
    the LL limit the same sequence exercises the LL slot reuse instead: rank 0's
    launch C may write slot (A & 1) only once rank 1 acknowledged launch A."""
    from paper_2604_00317_b200 import comm as C
    comm.set_config(pull=2)  # every registered sender grants pulls

    def mat(a10, a11, a00):
        m = [0] * (R * R)
        m[1 * R + 0], m[1 * R + 1], m[0] = a10, a11, a00
        return m

    mats = [mat(small, big, 0), mat(0, 0, 4096), mat(small, 0, 0)]
    bufs, handles = [], []
    for i, m in enumerate(mats):
        sc, sd, rc, rd = C.packed_displs(m, R, rank)
        send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
        recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
        for d in range(R):
            C.fill_payload(send[sd[d]:], 0, sc[d], 40 + i, rank, d)
        handles += [comm.register(send), comm.register(recv)]
        bufs.append((m, sc, sd, recv, rc, rd, send))
    _sync()
    for m, sc, sd, recv, rc, rd, send in bufs:  # no host sync between the launches
        comm.alltoallv(send, sc, sd, recv, rc, rd)
    _sync()
    comm.check_async()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for i, (m, sc, sd, recv, rc, rd, send) in enumerate(bufs):
        for s in range(R):
            C.check_payload(recv[rd[s]:], 0, rc[s], 40 + i, s, rank, bad)
    _sync()
    for h in handles:
        comm.deregister(h)
    comm.set_config(pull=0)
    return int(bad.item())


def w_ll(comm, rank, R):
    """Low-latency protocol for pairs <= ll_max (1 MiB, cut into 8 KiB pieces):
    odd sizes around the piece and pair thresholds next to normal pairs, unaligned packed offsets, six back-to-back
    launches without a host sync (slot parity + acknowledgements), a CUDA graph
    replaying an all-LL exchange, and the same traffic with LL disabled."""
    from paper_2604_00317_b200 import comm as C
    sizes = [1, 7, 8, 9, 8191, 8192, 8193, 40961, 65535, 65536, 65537, 262144, 262145, 1 << 20, (1 << 20) + 1,
             3 << 20, 3]

    def mat(shift):
        return [0 if s == d else sizes[(3 * s + 5 * d + shift) % len(sizes)] for s in range(R) for d in range(R)]

    out = []
    for ll_max in (1 << 20, 256 << 10, 0):
        comm.set_config(ll_max=ll_max)
        runs = []
        for i in range(6):
            m = mat(i % 2)
            sc, sd, rc, rd = C.packed_displs(m, R, rank)
            send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
            recv = torch.full((max(sum(rc), 16),), 0xEE, dtype=torch.uint8, device="cuda")
            for d in range(R):
                C.fill_payload(send[sd[d]:], 0, sc[d], 60 + i, rank, d)
            runs.append((sc, sd, rc, rd, send, recv))
        _sync()
        for sc, sd, rc, rd, send, recv in runs:  # no host sync in between
            comm.alltoallv(send, sc, sd, recv, rc, rd)
        _sync()
        comm.check_async()
        bad = torch.zeros(1, dtype=torch.int64, device="cuda")
        for i, (sc, sd, rc, rd, send, recv) in enumerate(runs):
            for src in range(R):
                C.check_payload(recv[rd[src]:], 0, rc[src], 60 + i, src, rank, bad)
            if recv.numel() > sum(rc):
                bad += int((recv[sum(rc):] != 0xEE).sum())
        _sync()
        out.append(int(bad.item()))
    comm.set_config(ll_max=1 << 20)
    # an all-LL exchange captured in a CUDA graph
    m = [0 if s == d else 1000 + 13 * s + d for s in range(R) for d in range(R)]
    sc, sd, rc, rd = C.packed_displs(m, R, rank)
    send = torch.empty(sum(sc), dtype=torch.uint8, device="cuda")
    recv = torch.zeros(sum(rc), dtype=torch.uint8, device="cuda")
    comm.alltoallv(send, sc, sd, recv, rc, rd)
    _sync()
    g = _capture(lambda: comm.alltoallv(send, sc, sd, recv, rc, rd))
    _barrier()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for i in range(4):
        for d in range(R):
            C.fill_payload(send[sd[d]:], 0, sc[d], 90 + i, rank, d)
        recv.zero_()
        _sync()
        g.replay()
        _sync()
        for src in range(R):
            C.check_payload(recv[rd[src]:], 0, rc[src], 90 + i, src, rank, bad)
    _sync()
    comm.check_async()
    out.append(int(bad.item()))
    return out


def w_ll_mismatch(comm, rank, R):
    """LL-sized pair whose receiver expects one byte less: the header's byte
    count turns it into an async error, not silent truncation."""
    n = 4096
    x = torch.zeros(n, dtype=torch.uint8, device="cuda")
    y = torch.zeros(n, dtype=torch.uint8, device="cuda")
    sc = [n if d != rank else 0 for d in range(R)]
    rc = [n - (1 if rank == 1 and s == 0 else 0) if s != rank else 0 for s in range(R)]
    try:
        comm.alltoallv(x, sc, [0] * R, y, rc, [0] * R)
        _sync()
    except Exception as e:  # host-side detection is acceptable too
        return "raised: " + str(e)[:60]
    return comm.async_error()


def w_sendrecv_mixed(comm, rank, R):
    """One group with sends to two different peers: an LL-sized message to the
    right neighbour, a normal-path one to the left, and a zero-byte one;
    several rounds back to back with different sizes."""
    from paper_2604_00317_b200 import comm as C
    right, left = (rank + 1) % R, (rank - 1) % R
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    if R == 2:  # one peer: an LL-sized message one way, a normal-path one back
        for it, (small, big) in enumerate([(3, (1 << 20) + 300001), (262144, 3 * MiB + 1)]):
            n_out, n_in = (small, big) if rank == 0 else (big, small)
            x = torch.empty(n_out, dtype=torch.uint8, device="cuda")
            C.fill_payload(x, 0, n_out, 500 + it, rank, 1 - rank)
            y = torch.zeros(n_in, dtype=torch.uint8, device="cuda")
            with C.group():
                comm.send(x, n_out, 1 - rank)
                comm.recv(y, n_in, 1 - rank)
            _sync()
            comm.check_async()
            C.check_payload(y, 0, n_in, 500 + it, 1 - rank, rank, bad)
        _sync()
        return int(bad.item())
    for it, (small, big) in enumerate([(3, 300001), (8192 + 5, 2 * MiB + 1), (262144, 262145)]):
        xs = torch.empty(small, dtype=torch.uint8, device="cuda")
        xb = torch.empty(big, dtype=torch.uint8, device="cuda")
        C.fill_payload(xs, 0, small, 300 + it, rank, right)
        C.fill_payload(xb, 0, big, 400 + it, rank, left)
        ys = torch.zeros(small, dtype=torch.uint8, device="cuda")
        yb = torch.zeros(big, dtype=torch.uint8, device="cuda")
        z = torch.zeros(16, dtype=torch.uint8, device="cuda")
        with C.group():
            comm.send(xs, small, right)
            comm.send(xb, big, left)
            comm.recv(ys, small, left)    # left neighbour's small message is for me
            comm.recv(yb, big, right)     # right neighbour's big message is for me
            if R > 3:
                comm.send(z, 0, (rank + 2) % R)
                comm.recv(z, 0, (rank - 2) % R)
        _sync()
        comm.check_async()
        C.check_payload(ys, 0, small, 300 + it, left, rank, bad)
        C.check_payload(yb, 0, big, 400 + it, right, rank, bad)
    _sync()
    return int(bad.item())


def w_moe_autograd(comm, rank, R):
    """Differentiable dispatch / combine through the nimble_b200::alltoallv_rows
    custom op: forward and the gradients of x and of the router weights match
    the same computation done locally (fp32)."""
    from paper_2604_00317_b200 import moe
    g = torch.Generator(device="cuda").manual_seed(200 + rank)
    T, H, k, E = 513, 64, 2, 4 * R
    x = torch.randn(T, H, device="cuda", generator=g, requires_grad=True)
    w = torch.rand(T, k, device="cuda", generator=g, requires_grad=True)
    hot = torch.rand(T, k, device="cuda", generator=g) < 0.6
    ids = torch.where(hot, torch.zeros_like(hot, dtype=torch.int64),
                      torch.randint(0, E, (T, k), device="cuda", generator=g))
    gout = torch.randn(T, H, device="cuda", generator=g)
    epr = E // R
    recv_x, recv_e, h = moe.dispatch(comm, x, ids, E)
    y = recv_x * (recv_e.to(torch.float32) + rank * epr + 1).unsqueeze(1)
    out = moe.combine(comm, y, h, w)
    (out * gout).sum().backward()
    _sync()
    comm.check_async()
    x2, w2 = x.detach().clone().requires_grad_(True), w.detach().clone().requires_grad_(True)
    ref = (x2.unsqueeze(1) * (ids.to(torch.float32) + 1).unsqueeze(2) * w2.unsqueeze(2)).sum(1)
    (ref * gout).sum().backward()
    ok = (torch.allclose(out, ref, rtol=1e-5, atol=1e-5) and torch.allclose(x.grad, x2.grad, rtol=1e-5, atol=1e-5)
          and torch.allclose(w.grad, w2.grad, rtol=1e-4, atol=1e-4))
    return bool(ok), sum(h.recv_counts)


def w_stress_ll(comm, rank, R):
    """40 launches back to back without a host sync, alternating three small
    skewed matrices whose pairs straddle the LL limit (some pairs LL, some on
    the post / pull / push path) and two receive buffers each, then every
    buffer's last delivery is verified."""
    import random
    from paper_2604_00317_b200 import comm as C
    from paper_2604_00317_b200 import planner as P
    rng = random.Random(11)  # same sequence on every rank
    pool = []
    for it, per_rank in enumerate((64 * 1024 + 5, 600 * 1024 + 1, 2 * MiB + 3)):
        m = P.gen_skewed_a2av(R, per_rank, 0.7, it % R)
        sc, sd, rc, rd = C.packed_displs(m, R, rank)
        send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
        for d in range(R):
            C.fill_payload(send[sd[d]:], 0, sc[d], 70 + it, rank, d)
        recvs = [torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda") for _ in range(2)]
        hs = [comm.register(send), comm.register(recvs[0])] if it != 1 else []
        pool.append((sc, sd, rc, rd, send, recvs, hs, 70 + it))
    _sync()
    plan = [(rng.randrange(3), rng.randrange(2)) for _ in range(40)]
    for k, (i, j) in enumerate(plan):
        if k % 10 == 0:
            comm.set_config(pull=rng.choice([0, 1, 2]))
        sc, sd, rc, rd, send, recvs, hs, seed = pool[i]
        comm.alltoallv(send, sc, sd, recvs[j], rc, rd)
    _sync()
    comm.check_async()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for i, (sc, sd, rc, rd, send, recvs, hs, seed) in enumerate(pool):
        for j in range(2):
            if (i, j) in plan:
                for s in range(R):
                    C.check_payload(recvs[j][rd[s]:], 0, rc[s], seed, s, rank, bad)
    _sync()
    for (sc, sd, rc, rd, send, recvs, hs, seed) in pool:
        for h in hs:
            comm.deregister(h)
    comm.set_config(pull=0)
    return int(bad.item())


def w_bench(comm, rank, R):
    return comm.bench_skewed(32 * MiB, 0.7, 0, warmup=1, iters=3)


def w_relay_split(comm, rank, R, nbytes):
    """c1 / c2: p2p 0 -> 1 on the mesh model.  Delivery is checked byte for
    byte, and the engine's per-kind device byte counters show the plan's
    split really crossed the relays: rank 0 pushes the direct flow and stages
    each relay flow into its relay's ring, every relay forwards exactly its
    flow to rank 1 (reference test_planner.cpp:96-111
    style goldens).  Also returns the slot-occupancy counters."""
    from paper_2604_00317_b200 import planner as P
    comm.set_config(fabric="alltoall", gpus_per_node=R)
    comm.stats(reset=True)
    m = P.gen_p2p(R, 0, 1, nbytes)
    bad, ok = _exchange_and_check(comm, rank, R, m, True, 23, host_check=nbytes <= 256 * MiB)
    st = comm.stats(reset=True)
    comm.set_config(fabric="nvswitch")
    return bad, ok, {k: st[k] for k in ("push", "stage", "forward", "pull", "drain")}


def w_check_detects_corruption(comm, rank, R):
    """The device checker counts exactly the bytes an exchange got wrong."""
    from paper_2604_00317_b200 import comm as C
    from paper_2604_00317_b200 import planner as P
    m = P.gen_skewed_a2av(R, 3 * MiB + 5, 0.7, 0)
    sc, sd, rc, rd = C.packed_displs(m, R, rank)
    send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
    recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
    for d in range(R):
        C.fill_payload(send[sd[d]:], 0, sc[d], 3, rank, d)
    comm.alltoallv(send, sc, sd, recv, rc, rd)
    _sync()
    src = (rank + 1) % R
    flips = [0, 1, rc[src] // 2, rc[src] - 1]
    for f in flips:
        recv[rd[src] + f] ^= 0x5A
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s in range(R):
        C.check_payload(recv[rd[s]:], 0, rc[s], 3, s, rank, bad)
    _sync()
    return int(bad.item()), len(set(flips))


ALL = _layouts(2, 4, 8)
SOME = _layouts(2, 8)


@pytest.mark.parametrize("layout", ALL)
@pytest.mark.parametrize("register", [True, False])
@pytest.mark.parametrize("per_rank,ratio", [(8 * MiB + 13, 0.7), (64 * MiB, 0.9), (1000, 0.5)])
def test_skewed_alltoallv(layout, per_rank, ratio, register):
    for r, (bad, ok) in _run(layout, "w_skewed", per_rank, ratio, register).items():
        assert bad == 0 and ok, r


@pytest.mark.parametrize("layout", _layouts(3, 5, 7, proc_min=3))
def test_ragged_matrices_odd_rank_counts(layout):
    for r, oks in _run(layout, "w_ragged_fuzz", [101, 202, 303]).items():
        assert all(oks), (r, oks)


@pytest.mark.parametrize("layout", ALL)
def test_pull_modes_all_registration_combinations(layout):
    for r, res in _run(layout, "w_pull_modes").items():
        assert all(bad == 0 and ok for bad, ok in res), (r, res)


@pytest.mark.parametrize("layout", ALL)
def test_irregular_c4_sizes_registered_and_staged(layout):
    for r, res in _run(layout, "w_irregular").items():
        assert all(bad == 0 and ok for bad, ok in res), (r, res)


@pytest.mark.parametrize("layout", SOME)
def test_repeated_mixed_exchanges(layout):
    for r, res in _run(layout, "w_repeat_mixed").items():
        assert all(bad == 0 and ok for bad, ok in res), (r, res)


@pytest.mark.parametrize("layout", ALL)
def test_stress_back_to_back_exchanges(layout):
    assert all(v == 0 for v in _run(layout, "w_stress_back_to_back").values())


@pytest.mark.parametrize("layout", SOME)
def test_sendrecv_group_ring(layout):
    assert all(v == 0 for v in _run(layout, "w_sendrecv_ring").values())


@pytest.mark.parametrize("layout", _layouts(3, 4, proc_min=3))
def test_relay_routes_execute_bit_exact(layout):
    R = layout[1]
    for r, ((bad, ok), relays, mism) in _run(layout, "w_relay", 256 * MiB).items():
        assert bad == 0 and ok and mism == 0, r
        assert relays == R - 2  # one relay flow per intermediate GPU


C1_DIRECT, C1_RELAY = 33554432, 33554432                  # c1: 64 MiB on mesh3
C2_DIRECT, C2_RELAY = 360710144, 356515840                # c2: 1 GiB on mesh4: direct + 2 relays


@pytest.mark.parametrize("layout", _layouts(3, proc_min=3, proc_max=3))
def test_c1_relay_split_crosses_the_relay(layout):
    out = _run(layout, "w_relay_split", 64 * MiB)
    for r, (bad, ok, st) in out.items():
        assert bad == 0 and ok, r
    st0, st2 = out[0][2], out[2][2]
    assert st0["push"][1] == C1_DIRECT and st0["stage"][2] == C1_RELAY and st0["pull"] == [0, 0, 0]
    assert st2["forward"][1] == C1_RELAY and sum(st2["push"]) == 0
    assert sum(out[1][2]["push"]) + sum(out[1][2]["stage"]) == 0  # rank 1 only receives


@pytest.mark.parametrize("layout", _layouts(4, proc_min=4, proc_max=4))
def test_c2_two_relays_split(layout):
    out = _run(layout, "w_relay_split", 1 << 30)
    for r, (bad, ok, st) in out.items():
        assert bad == 0 and ok, r
    st0 = out[0][2]
    assert st0["push"][1] == C2_DIRECT and st0["stage"][2] == C2_RELAY and st0["stage"][3] == C2_RELAY
    for v in (2, 3):
        assert out[v][2]["forward"][1] == C2_RELAY, v
    assert C2_DIRECT + 2 * C2_RELAY == 1 << 30


@pytest.mark.parametrize("layout", SOME)
def test_checker_counts_corrupted_bytes(layout):
    for r, (bad, want) in _run(layout, "w_check_detects_corruption").items():
        assert bad == want, (r, bad, want)


@pytest.mark.parametrize("layout", SOME)
def test_count_mismatch_is_an_error_not_a_hang(layout):
    res = _run(layout, "w_mismatch")
    assert any(v not in (0, "0") for v in res.values()), res


@pytest.mark.parametrize("layout", _layouts(2, 4))
def test_moe_dispatch_combine(layout):
    res = _run(layout, "w_moe")
    assert all(ok for ok, _ in res.values()), res
    assert res[0][1] > max(n for r, (_, n) in res.items() if r != 0)  # rank 0 holds the hot expert


@pytest.mark.parametrize("layout", ALL)
def test_cuda_graph_capture_and_replay(layout):
    for r, bads in _run(layout, "w_graph").items():
        assert bads == [0] * 6, (r, bads)  # 5 replays, then one after cache churn + a deregistration


@pytest.mark.parametrize("layout", SOME)
def test_bench_entry_point(layout):
    for r, b in _run(layout, "w_bench").items():
        assert b["mismatches"] == 0 and b["gbps_effective"] > 0 and b["bound_seconds"] > 0


@pytest.mark.multigpu
@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_comm_init_all_single_process_grouped():
    """nimbleCommInitAll: every GPU in this process, one grouped call per step
    (NCCL's single-process pattern), registered and unregistered receives,
    mesh model (row allgather inside the clique) included."""
    _init_all_grouped(list(range(min(_ngpus(), 4))))


@pytest.mark.parametrize("R", [2, 4])
def test_comm_init_all_repeated_device(R):
    """nimbleCommInitAll([0] * R): R co-resident ranks driven from ONE thread
    with grouped calls, one stream per rank."""
    _init_all_grouped([0] * R)


def _init_all_grouped(devices):
    from paper_2604_00317_b200 import comm as C
    from paper_2604_00317_b200 import planner as P
    R = len(devices)
    comms = C.Comm.init_all(devices)
    streams = []
    for c in comms:
        with torch.cuda.device(c.device):
            streams.append(torch.cuda.Stream())
    try:
        for fabric, register, per_rank in (("nvswitch", True, 3 * MiB + 1), ("nvswitch", False, 3 * MiB + 1),
                                           ("alltoall", True, 0), ("nvswitch", False, 100 * 1024 + 3)):  # last: LL
            for c in comms:
                with torch.cuda.device(c.device):
                    c.set_config(fabric=fabric, gpus_per_node=R)
            m = P.gen_p2p(R, 0, 1, 96 * MiB) if fabric == "alltoall" else P.gen_skewed_a2av(R, per_rank, 0.7, 0)
            bufs = []
            for c in comms:
                with torch.cuda.device(c.device):
                    sc, sd, rc, rd = C.packed_displs(m, R, c.rank)
                    send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
                    recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
                    for d in range(R):
                        C.fill_payload(send[sd[d]:], 0, sc[d], 77, c.rank, d)
                    torch.cuda.synchronize()
                    hs = [c.register(send), c.register(recv)] if register else []
                    bufs.append((c, send, recv, sc, sd, rc, rd, hs))
            with C.group():
                for (c, send, recv, sc, sd, rc, rd, hs), st in zip(bufs, streams):
                    with torch.cuda.device(c.device):
                        c.alltoallv(send, sc, sd, recv, rc, rd, stream=st)
            for (c, send, recv, sc, sd, rc, rd, hs), st in zip(bufs, streams):
                with torch.cuda.device(c.device):
                    st.synchronize()
                    c.check_async()
                    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
                    for s in range(R):
                        C.check_payload(recv[rd[s]:], 0, rc[s], 77, s, c.rank, bad)
                    torch.cuda.synchronize()
                    assert int(bad.item()) == 0, (fabric, register, c.rank)
                    for h in hs:
                        c.deregister(h)
    finally:
        for c in comms:
            with torch.cuda.device(c.device):
                c.destroy()


@pytest.mark.parametrize("layout", _layouts(2, proc_max=2))
@pytest.mark.parametrize("small", [(1 << 20) + 300 * 1024 + 3, 4096 + 3])  # pull path (> ll_max), LL path
def test_receiver_two_launches_ahead_of_sender(layout, small):
    out = _run(layout, "w_overtake", 4 << 30, small)
    assert all(v == 0 for v in out.values()), out


@pytest.mark.parametrize("layout", ALL)
def test_low_latency_protocol_small_pairs(layout):
    out = _run(layout, "w_ll")
    assert all(v == [0, 0, 0, 0] for v in out.values()), out  # three ll_max settings + the graph


@pytest.mark.parametrize("layout", _layouts(2, proc_max=2))
def test_low_latency_size_mismatch_is_an_error(layout):
    out = _run(layout, "w_ll_mismatch")
    assert out[1] != 0, out  # the receiver that expected fewer bytes reports it


@pytest.mark.parametrize("layout", _layouts(2, 3, 8))
def test_sendrecv_group_mixed_sizes_and_peers(layout):
    out = _run(layout, "w_sendrecv_mixed")
    assert all(v == 0 for v in out.values()), out


@pytest.mark.parametrize("layout", _layouts(2, 4))
def test_moe_custom_op_forward_and_gradients(layout):
    res = _run(layout, "w_moe_autograd")
    assert all(ok for ok, _ in res.values()), res


@pytest.mark.parametrize("layout", ALL)
def test_stress_ll_and_normal_pairs_back_to_back(layout):
    out = _run(layout, "w_stress_ll")
    assert all(v == 0 for v in out.values()), out


def w_sendrecv_multi(comm, rank, R):
    """NCCL group semantics: several sends to one peer and several receives
    from one peer in one group, matched in issue order (odd sizes, a zero-byte
    operation in between, one part above the LL limit), next to a plain pair;
    each receive buffer holds exactly its part of the pair's payload."""
    from paper_2604_00317_b200 import comm as C
    right, left = (rank + 1) % R, (rank - 1) % R
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for it, sizes in enumerate([[3, 0, 70001, 8192], [(1 << 20) + 5, 77, 2 * MiB + 3], [1, 2, 3, 4, 5]]):
        xs, ys, off = [], [], 0
        for n in sizes:
            x = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
            C.fill_payload(x, off, n, 700 + it, rank, right)
            xs.append((x, n, off))
            ys.append((torch.zeros(max(n, 1), dtype=torch.uint8, device="cuda"), n, off))
            off += n
        one = 5 * MiB + 1
        z = torch.empty(one, dtype=torch.uint8, device="cuda")
        C.fill_payload(z, 0, one, 800 + it, rank, (rank + 2) % R)
        zr = torch.zeros(one, dtype=torch.uint8, device="cuda")
        with C.group():
            for x, n, _ in xs:
                comm.send(x, n, right)
            for y, n, _ in ys:
                comm.recv(y, n, left)
            if R > 2:
                comm.send(z, one, (rank + 2) % R)
                comm.recv(zr, one, (rank - 2) % R)
        _sync()
        comm.check_async()
        for y, n, o in ys:
            C.check_payload(y, o, n, 700 + it, left, rank, bad)
        if R > 2:
            C.check_payload(zr, 0, one, 800 + it, (rank - 2) % R, rank, bad)
    _sync()
    return int(bad.item())


@pytest.mark.parametrize("layout", _layouts(2, 4))
def test_sendrecv_several_ops_per_peer(layout):
    out = _run(layout, "w_sendrecv_multi")
    assert all(v == 0 for v in out.values()), out


def w_moe_counts(comm, rank, R):
    """The MoE dispatch's count exchange alone (alltoall of one int64 per
    peer) and its row exchange sizes: returns (count_out, count_in)."""
    from paper_2604_00317_b200.moe import MoEDispatcher
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    T, H, k, E = 777, 96, 2, 4 * R
    x = torch.randn(T, H, device="cuda", generator=g)
    hot = torch.rand(T, k, device="cuda", generator=g) < 0.6
    ids = torch.where(hot, torch.zeros_like(hot, dtype=torch.int64),
                      torch.randint(0, E, (T, k), device="cuda", generator=g))
    disp = MoEDispatcher(comm, E, H, dtype=torch.float32, max_tokens=1024, topk=k)
    try:
        recv_x, recv_e, h = disp.dispatch(x, ids)
        _sync()
        comm.check_async()
        return list(h.send_counts), list(h.recv_counts)
    finally:
        disp.close()


@pytest.mark.parametrize("layout", _layouts(2, 4))
def test_moe_count_exchange_consistent(layout):
    out = _run(layout, "w_moe_counts")
    R = len(out)
    for r in range(R):
        for s in range(R):
            assert out[r][1][s] == out[s][0][r], (r, s, out)


def w_count_variants(comm, rank, R, variant, reps):
    """Debug aid: the MoE count exchange (8-byte LL pairs + an 8-byte self
    copy) `reps` times, with (variant) nothing else / torch kernels between
    exchanges / five registered windows.  Returns the reps whose counts came
    back wrong; raises on an async error."""
    hs = []
    if variant == "reg":
        bufs = [torch.empty(1 << 20, dtype=torch.uint8, device="cuda") for _ in range(5)]
        hs = [comm.register(b) for b in bufs]
    out = torch.full((R,), rank + 1, dtype=torch.int64, device="cuda")
    wrong = []
    for i in range(reps):
        if variant == "torch":
            x = torch.rand(20000, device="cuda")
            o = torch.argsort(x, stable=True)
            torch.bincount(o % 7, minlength=R)
        inn = torch.zeros(R, dtype=torch.int64, device="cuda")
        out.fill_(rank + 1 + i)
        comm.alltoall(out, inn, 8)
        _sync()  # GIL released while waiting: tolist() would block holding it
        got = inn.tolist()
        comm.check_async()  # fail at the first bad exchange (its trace is the last launch's)
        if got != [s + 1 + i for s in range(R)]:
            wrong.append((i, got))
    _sync()
    comm.check_async()
    for h in hs:
        comm.deregister(h)
    return wrong


@pytest.mark.parametrize("variant", ["plain", "torch", "reg"])
@pytest.mark.parametrize("layout", _layouts(4, proc=False))
def test_count_exchange_variants(layout, variant):
    out = _run(layout, "w_count_variants", variant, 30)
    assert all(v == [] for v in out.values()), out
