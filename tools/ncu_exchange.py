"""Minimal multi-rank exchange for Nsight Compute captures (no gloo, no NCCL).

  torchrun --nproc-per-node N --no-python bash tools/rank0_ncu.sh OUT.csv SKIP COUNT -- \
      tools/ncu_exchange.py [--per-rank-mib 256] [--ratio 0.7] [--calls 8] [--case c3|c5]

Rank 0 (which may run under ncu, slow to start) writes the communicator id
to a file the other ranks wait for; everything after that goes through the
library's own bootstrap and exchanges.  Runs `calls` exchanges of the
BASELINE matrix on registered windows, then checks delivery; prints one
line per rank.
"""
import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-rank-mib", type=int, default=256)
    ap.add_argument("--ratio", type=float, default=0.7)
    ap.add_argument("--calls", type=int, default=8)
    ap.add_argument("--case", default="c3")
    args = ap.parse_args()
    if os.environ.get("NCU_DUMP_AFTER_S"):  # where a rank hangs (stack dump to stderr)
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["NCU_DUMP_AFTER_S"]), repeat=True)
    rank, R = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    os.environ.setdefault("NIMBLE_BOOTSTRAP_TIMEOUT_MS", "600000")
    path = os.path.join(ROOT, "gpurun_out", f".ncu_uid_{os.environ.get('MASTER_PORT', '0')}_{os.environ.get('TORCHELASTIC_RUN_ID', '')}")
    if rank == 0:
        if os.path.exists(path):
            os.remove(path)
        uid = C.unique_id()
        with open(path + ".tmp", "wb") as f:
            f.write(uid)
        os.replace(path + ".tmp", path)
    else:
        while not os.path.exists(path):
            time.sleep(0.05)
        time.sleep(0.05)
        with open(path, "rb") as f:
            uid = f.read()
    comm = C.Comm.init_rank(R, uid, rank)
    ratio = 1.0 / (R - 1) if args.case == "c5" else args.ratio
    m = P.gen_skewed_a2av(R, args.per_rank_mib * MiB, ratio, 0)
    sc, sd, rc, rd = C.packed_displs(m, R, rank)
    send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
    recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
    for d in range(R):
        C.fill_payload(send[sd[d]:], 0, sc[d], 1, rank, d)
    hs = [comm.register(recv), comm.register(send)]
    for k in range(args.calls):
        comm.alltoallv(send, sc, sd, recv, rc, rd)
        print(f"rank {rank}: call {k} enqueued", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    print(f"rank {rank}: synchronized", file=sys.stderr, flush=True)
    comm.check_async()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s in range(R):
        C.check_payload(recv[rd[s]:], 0, rc[s], 1, s, rank, bad)
    torch.cuda.synchronize()
    print(f"rank {rank}: {args.calls} exchanges, case {args.case} ratio {ratio:.3f} {args.per_rank_mib} MiB/rank, "
          f"ingress {sum(rc)} egress {sum(sc)} bytes, mismatched {int(bad.item())}", flush=True)
    for h in hs:
        comm.deregister(h)
    comm.destroy()
    if rank == 0:
        os.remove(path)


if __name__ == "__main__":
    main()
