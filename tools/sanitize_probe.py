"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
  local   -- the 1-GPU emulated exchange (one engine launch, no flags)
  comm1   -- a 1-rank communicator (posts, epilogue, LL off)
  thread2 -- 2 co-resident ranks on one GPU (the full cross-rank protocol;
             needs the sanitizer to let kernels of two streams run at once)
Each verifies delivery and prints one line; exit code 0 only if bit-exact."""
import os
import sys
import threading

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def local():
    R = 8
    m = P.gen_skewed_a2av(R, MiB + 4099, 0.7, 0)
    sends, recvs = [], []
    for s in range(R):
        sc, sd, _, _ = C.packed_displs(m, R, s)
        t = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
        for d in range(R):
            C.fill_payload(t[sd[d]:], 0, sc[d], 1, s, d)
        sends.append(t)
    for d in range(R):
        _, _, rc, _ = C.packed_displs(m, R, d)
        recvs.append(torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda"))
    C.exchange_local(sends, recvs, m, 16)
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for d in range(R):
        _, _, rc, rd = C.packed_displs(m, R, d)
        for s in range(R):
            C.check_payload(recvs[d][rd[s]:], 0, rc[s], 1, s, d, bad)
    torch.cuda.synchronize()
    return int(bad.item())


def run_ranks(R, per_rank, register):
    uid = C.unique_id()
    out = [None] * R

    def th(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            comm = C.Comm.init_rank(R, uid, r)
            m = P.gen_skewed_a2av(R, per_rank, 0.7, 0) if R > 1 else [per_rank]
            sc, sd, rc, rd = C.packed_displs(m, R, r)
            send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
            recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
            for d in range(R):
                C.fill_payload(send[sd[d]:], 0, sc[d], 2, r, d)
            hs = [comm.register(send), comm.register(recv)] if register else []
            for _ in range(2):
                comm.alltoallv(send, sc, sd, recv, rc, rd)
            st.synchronize()
            comm.check_async()
            bad = torch.zeros(1, dtype=torch.int64, device="cuda")
            for s in range(R):
                C.check_payload(recv[rd[s]:], 0, rc[s], 2, s, r, bad)
            st.synchronize()
            out[r] = int(bad.item())
            for h in hs:
                comm.deregister(h)
            comm.destroy()

    ts = [threading.Thread(target=th, args=(r,)) for r in range(R)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    return sum(x if x is not None else 1 for x in out)


if __name__ == "__main__":
    os.environ.setdefault("NIMBLE_TIMEOUT_MS", "20000")
    what = sys.argv[1]
    torch.cuda.set_device(0)
    if what == "local":
        bad = local()
    elif what == "comm1":
        bad = run_ranks(1, 3 * MiB + 5, False)
    else:
        bad = run_ranks(2, MiB + 77, True) + run_ranks(2, 600 * 1024, False)
    print(f"{what}: mismatched bytes {bad}")
    sys.exit(1 if bad else 0)
