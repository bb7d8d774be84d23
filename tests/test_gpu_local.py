"""GPU parity of the forwarding engine on one B200 (through the C ABI).

The oracle for delivery is oracle/cpu_exchange.c's orc_alltoallv (host
restatement of all-to-allv semantics); every comparison is bit-exact.
"""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

MiB = 1 << 20


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _oracle_exchange(m, R, host_send):
    from oracle import ref
    want = [np.zeros(max(sum(m[s * R + d] for s in range(R)), 1), dtype=np.uint8) for d in range(R)]
    mat = (ctypes.c_uint64 * (R * R))(*m)
    sp = (ctypes.c_void_p * R)(*[h.ctypes.data for h in host_send])
    rp = (ctypes.c_void_p * R)(*[w.ctypes.data for w in want])
    ref.cpu_lib().orc_alltoallv(R, mat, sp, rp)
    return want


def _run_local(m, R, seed=0, ctas=0):
    from paper_2604_00317_b200 import comm as C
    rng = np.random.default_rng(seed)
    host_send = [rng.integers(0, 256, max(sum(m[s * R:(s + 1) * R]), 1), dtype=np.uint8) for s in range(R)]
    sends = [torch.from_numpy(h).cuda() for h in host_send]
    recvs = [torch.full((max(sum(m[x * R + d] for x in range(R)), 1),), 0xEE, dtype=torch.uint8, device="cuda")
             for d in range(R)]
    C.exchange_local(sends, recvs, m, ctas)
    torch.cuda.synchronize()
    want = _oracle_exchange(m, R, host_send)
    for d in range(R):
        n = sum(m[x * R + d] for x in range(R))
        got = recvs[d].cpu().numpy()
        assert np.array_equal(got[:n], want[d][:n]), f"receiver {d}: {(got[:n] != want[d][:n]).sum()} bytes differ"
    return recvs


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


@pytest.mark.parametrize("per_rank,ratio", [(12, 0.5), (1000, 0.7), (MiB + 4099, 0.7), (3 * MiB + 1, 0.0),
                                            (2 * MiB + 7, 1.0), (4 * MiB, 1 / 7)])
def test_local_skewed_matches_oracle(per_rank, ratio):
    from paper_2604_00317_b200 import planner as P
    m = P.gen_skewed_a2av(8, per_rank, ratio, 0)
    _run_local(m, 8, seed=per_rank)


@pytest.mark.parametrize("total", [1024, 4096, 65536, 1 << 20, 16 << 20, 64 << 20])
def test_local_irregular_c4_sizes(total):  # c4: gen_irregular(8, T, 0.5, seed=1)
    from paper_2604_00317_b200 import planner as P
    _run_local(P.gen_irregular(8, total, 0.5, 1), 8, seed=total)


def test_local_edge_matrices():
    from paper_2604_00317_b200 import planner as P
    _run_local([0] * 16, 4)                                # empty exchange
    _run_local(P.gen_p2p(2, 0, 1, 1), 2)                   # one byte
    _run_local(P.gen_p2p(3, 2, 0, 5 * MiB + 3), 3)         # one pair
    _run_local(P.gen_stencil_1d(5, 777777), 5)             # ragged, sparse
    _run_local(P.gen_aggregator(6, [1, 4], 3 * MiB + 5), 6)
    m = P.gen_irregular(8, 8 * MiB + 123, 0.5, 9)
    for i in range(8):
        m[i * 8 + i] = 4096 + i                            # self segments
    _run_local(m, 8)


@pytest.mark.parametrize("ctas", [1, 3, 148, 500])
def test_local_grid_sizes(ctas):
    from paper_2604_00317_b200 import planner as P
    _run_local(P.gen_skewed_a2av(8, 2 * MiB + 33, 0.7, 0), 8, ctas=ctas)


def test_local_full_size_c3_payload_and_idempotence():
    """c3 at 256 MiB/rank: size-independent checks (payload function, two runs
    agree, byte sums conserved)."""
    from paper_2604_00317_b200 import comm as C
    from paper_2604_00317_b200 import planner as P
    R = 8
    m = P.gen_skewed_a2av(R, 256 * MiB, 0.7, 0)
    sends, recvs = [], []
    for s in range(R):
        sends.append(torch.empty(sum(m[s * R:(s + 1) * R]), dtype=torch.uint8, device="cuda"))
        sc, sd, _, _ = C.packed_displs(m, R, s)
        for d in range(R):
            C.fill_payload(sends[s][sd[d]:], 0, sc[d], 3, s, d)
    for d in range(R):
        recvs.append(torch.zeros(sum(m[x * R + d] for x in range(R)), dtype=torch.uint8, device="cuda"))
    C.exchange_local(sends, recvs, m)
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for d in range(R):
        _, _, rc, rd = C.packed_displs(m, R, d)
        for s in range(R):
            C.check_payload(recvs[d][rd[s]:], 0, rc[s], 3, s, d, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 0
    first = [r.clone() for r in recvs]
    C.exchange_local(sends, recvs, m)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(first, recvs))
    total_in = sum(int(s.to(torch.int64).sum()) for s in sends)
    total_out = sum(int(r.to(torch.int64).sum()) for r in recvs)
    assert total_in == total_out


def test_single_rank_comm_self_segment():
    """A 1-rank communicator: the self segment is a local copy, registered or not."""
    from paper_2604_00317_b200 import comm as C
    c = C.Comm.init_rank(1, C.unique_id(), 0)
    try:
        x = torch.randint(0, 256, (3 * MiB + 5,), dtype=torch.uint8, device="cuda")
        y = torch.zeros_like(x)
        c.alltoallv(x, [x.numel()], [0], y, [x.numel()], [0])
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        h = c.register(y)
        y.zero_()
        c.alltoall(x, y, x.numel())
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        c.deregister(h)
        c.check_async()
    finally:
        c.destroy()


def test_single_rank_chained_exchanges_see_user_kernels():
    """Exchange chaining (engine.cu): back-to-back exchanges chain on the
    epoch word, and an exchange whose predecessor on the stream is a user
    kernel must still see that kernel's writes.  A 1-rank comm launches with
    PDL, so both paths run here: every other step a torch kernel rewrites the
    send buffer right before the exchange, and the result is checked on the
    device after each step (no host sync in between)."""
    from paper_2604_00317_b200 import comm as C
    c = C.Comm.init_rank(1, C.unique_id(), 0)
    try:
        n = 5 * MiB + 3
        x = torch.zeros(n, dtype=torch.uint8, device="cuda")
        y = torch.zeros_like(x)
        hx, hy = c.register(x), c.register(y)
        c.alltoallv(x, [n], [0], y, [n], [0])  # warm-up: schedule cached
        bad = torch.zeros(1, dtype=torch.int64, device="cuda")
        for k in range(60):
            if k % 2 == 0:
                x.fill_(k & 0xFF)  # a user kernel right before the exchange
            c.alltoallv(x, [n], [0], y, [n], [0])
            c.alltoallv(x, [n], [0], y, [n], [0])  # chained on the previous exchange
            bad += (y != x).sum()
        torch.cuda.synchronize()
        c.check_async()
        assert int(bad.item()) == 0
        c.deregister(hx)
        c.deregister(hy)
    finally:
        c.destroy()


def test_two_comms_alternating_on_one_stream():
    """Two comms' exchanges interleaved on one stream never chain on each
    other (each launch's predecessor is the other comm's exchange, so it
    waits for that grid): delivery stays exact and nothing hangs."""
    from paper_2604_00317_b200 import comm as C
    a = C.Comm.init_rank(1, C.unique_id(), 0)
    b = C.Comm.init_rank(1, C.unique_id(), 0)
    try:
        n = 3 * MiB + 11
        xa = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
        xb = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
        ya, yb = torch.zeros_like(xa), torch.zeros_like(xb)
        bad = torch.zeros(1, dtype=torch.int64, device="cuda")
        for k in range(40):
            a.alltoallv(xa, [n], [0], ya, [n], [0])
            b.alltoallv(ya if k % 2 else xb, [n], [0], yb, [n], [0])  # b reads what a just wrote, half the time
            bad += (ya != xa).sum() + (yb != (ya if k % 2 else xb)).sum()
            xa.add_(1)
        torch.cuda.synchronize()
        a.check_async()
        b.check_async()
        assert int(bad.item()) == 0
    finally:
        a.destroy()
        b.destroy()


def test_comm_init_all_single_device():
    from paper_2604_00317_b200 import comm as C
    comms = C.Comm.init_all([0])
    try:
        assert comms[0].nranks == 1 and comms[0].rank == 0 and comms[0].device == 0
        x = torch.arange(1000, dtype=torch.int32, device="cuda").view(torch.uint8)
        y = torch.zeros_like(x)
        with C.group():
            comms[0].send(x, x.numel(), 0)
            comms[0].recv(y, y.numel(), 0)
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    finally:
        comms[0].destroy()


def test_payload_fill_matches_oracle():
    from oracle import ref
    from paper_2604_00317_b200 import comm as C
    n = 100003
    for first in (0, 5, 8, 13):
        t = torch.zeros(n, dtype=torch.uint8, device="cuda")
        C.fill_payload(t, first, n, 77, 3, 5)
        want = np.zeros(n, dtype=np.uint8)
        ref.cpu_lib().orc_fill(want.ctypes.data, first, n, 77, 3, 5)
        assert np.array_equal(t.cpu().numpy(), want)


def test_comm_config_validation():
    from paper_2604_00317_b200 import comm as C
    from paper_2604_00317_b200._lib import NimbleError
    c = C.Comm.init_rank(1, C.unique_id(), 0)
    try:
        cfg = c.config()
        assert cfg.fabric == 1 and cfg.pipe_chunk == 64 << 10 and cfg.p2p_buffer == 10 << 20 and cfg.pull == 0
        assert cfg.push_chunk == 0 and cfg.direct_chunk == 0
        with pytest.raises(NimbleError):
            c.set_config(fabric="alltoall", gpus_per_node=4)      # mesh model needs one GPU per rank
        with pytest.raises(NimbleError):
            c.set_config(pipe_chunk=64 << 10, p2p_buffer=32 << 20)  # 512 slots > 256
        with pytest.raises(NimbleError):
            c.set_config(pipe_chunk=1 << 20, p2p_buffer=512 << 10)  # buffer holds no chunk
        c.set_config(pipe_chunk=512 << 10, p2p_buffer=10 << 20)     # the reference's geometry is valid
        assert c.config().pipe_chunk == 512 << 10
    finally:
        c.destroy()
