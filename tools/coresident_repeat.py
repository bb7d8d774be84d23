"""Repeat one co-resident (thread-mode) GPU test worker many times on GPU 0.

  python tools/coresident_repeat.py w_moe 4 20 [args...]

Runs tests/test_gpu_comm.py's worker `fn` as R ranks in one process (the same
harness the `-m gpu` tests use) `reps` times and prints one line per rep.
NIMBLE_LAUNCH_LOG=1 (inherited by the server) logs every engine launch on
stderr, so a failing rep can be compared launch by launch across ranks.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import test_gpu_comm as T  # noqa: E402


def w_moe_timed(comm, rank, R):
    """tests' w_moe with a host timeline (CLOCK_REALTIME ns, the clock the
    engine's %globaltimer trace follows) of every step.  Returns the
    timeline, the async error and the last launch's device trace instead of
    raising, so every rank's view of a failing rep is printed."""
    import torch
    from paper_2604_00317_b200.moe import MoEDispatcher
    tl = []

    def mark(what):
        tl.append((what, time.time_ns()))

    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    T, H, k, E = 777, 96, 2, 4 * R
    x = torch.randn(T, H, device="cuda", generator=g)
    hot = torch.rand(T, k, device="cuda", generator=g) < 0.6
    ids = torch.where(hot, torch.zeros_like(hot, dtype=torch.int64),
                      torch.randint(0, E, (T, k), device="cuda", generator=g))
    w = torch.rand(T, k, device="cuda", generator=g)
    mark("inputs")
    disp = MoEDispatcher(comm, E, H, dtype=torch.float32, max_tokens=1024, topk=k)
    mark("dispatcher")
    orig, orig_a2a = comm.alltoallv, comm.alltoall
    try:
        def logged(*a, **kw):
            mark("a2av>")
            orig(*a, **kw)
            mark("a2av<")

        def logged_a2a(*a, **kw):
            mark("a2a>")
            orig_a2a(*a, **kw)
            mark("a2a<")
        comm.alltoallv, comm.alltoall = logged, logged_a2a
        recv_x, recv_e, h = disp.dispatch(x, ids)
        mark("dispatched")
        y = recv_x * (recv_e.to(torch.float32) + rank * disp.experts_per_rank + 1).unsqueeze(1)
        mark("expert")
        # combine, step by step
        m = sum(h.recv_counts)
        disp.recv_buf[:m].copy_(y)
        mark("c.copy")
        sb = [c * disp.row for c in h.recv_counts]
        rb = [c * disp.row for c in h.send_counts]
        comm.alltoallv(disp.recv_buf, sb, disp._displs(sb), disp.back_buf, rb, disp._displs(rb))
        n = h.num_tokens * h.topk
        back = disp.back_buf[:n]
        mark("c.back")
        wr = w.reshape(-1)[h.order]
        mark("c.index")
        back = back * wr.to(back.dtype).unsqueeze(1)
        mark("c.mul")
        out = torch.zeros(h.num_tokens, disp.hidden, dtype=disp.dtype, device=back.device)
        mark("c.zeros")
        out.index_add_(0, h.order // h.topk, back)
        mark("c.index_add")
        torch.cuda.current_stream().synchronize()
        mark("synced")
        return {"err": comm.async_error(), "trace": comm.debug_trace()[:7], "timeline": tl}
    finally:
        comm.alltoallv, comm.alltoall = orig, orig_a2a
        disp.close()


def main():
    fn, R, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    args = [int(a) if a.lstrip("-").isdigit() else a for a in sys.argv[4:]]
    fails = 0
    for i in range(reps):
        t0 = time.time()
        try:
            out = T._threads(fn, R, *args)
            print(f"rep {i}: ok {time.time() - t0:.2f}s {out}", flush=True)
        except BaseException as e:  # pytest.fail raises a BaseException subclass
            fails += 1
            print(f"rep {i}: FAIL {time.time() - t0:.2f}s {str(e)[:3000]}", flush=True)
            print(f"=== rep {i} failed", file=sys.stderr, flush=True)
    for r in list(T._SERVERS):
        T._stop(r)
    print(f"{fn} R={R}: {fails} of {reps} failed")


if __name__ == "__main__":
    main()
