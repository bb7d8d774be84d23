"""One process drives N GPUs (nimbleCommInitAll) for Nsight Compute: the
exchanges of all ranks are launched by one thread at each GroupEnd, rank 0
first.  Profile the LAST launch of a group (the other ranks' kernels are
already running on their GPUs, so the profiled one can finish):

  ncu --metrics ... -k regex:exchange_kernel --launch-skip 2N-1 --launch-count 1 \
      python tools/ncu_clique.py [--gpus N] [--per-rank-mib 256] [--ratio 0.7] [--groups 2]

With `--groups 2` the profiled launch is the final one, so no later launch
has to run under ncu's serialization.  The hot rank is rank 0; to profile
it last, pass --hot N-1 (the matrix is permuted so rank N-1 is the hotspot).
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--per-rank-mib", type=int, default=256)
    ap.add_argument("--ratio", type=float, default=0.7)
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--hot", type=int, default=0)
    args = ap.parse_args()
    R = args.gpus
    comms = C.Comm.init_all(list(range(R)))
    base = P.gen_skewed_a2av(R, args.per_rank_mib * MiB, args.ratio, 0)
    perm = [(r - args.hot) % R for r in range(R)]  # rank `hot` plays the generator's rank 0
    m = [base[perm[s] * R + perm[d]] for s in range(R) for d in range(R)]
    bufs, lay, streams = [], [], []
    for r in range(R):
        torch.cuda.set_device(r)
        sc, sd, rc, rd = C.packed_displs(m, R, r)
        send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device=r)
        recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device=r)
        for d in range(R):
            C.fill_payload(send[sd[d]:], 0, sc[d], 1, r, d)
        bufs.append((send, recv, comms[r].register(recv), comms[r].register(send)))
        lay.append((sc, sd, rc, rd))
        streams.append(torch.cuda.Stream(device=r))
    for r in range(R):
        torch.cuda.synchronize(r)
    for _ in range(args.groups):
        with C.group():
            for r in range(R):
                sc, sd, rc, rd = lay[r]
                comms[r].alltoallv(bufs[r][0], sc, sd, bufs[r][1], rc, rd, streams[r])
    for r in range(R):
        torch.cuda.synchronize(r)
    bad = 0
    for r in range(R):
        torch.cuda.set_device(r)
        comms[r].check_async()
        sc, sd, rc, rd = lay[r]
        cnt = torch.zeros(1, dtype=torch.int64, device=r)
        for s in range(R):
            C.check_payload(bufs[r][1][rd[s]:], 0, rc[s], 1, s, r, cnt)
        torch.cuda.synchronize(r)
        bad += int(cnt.item())
    print(f"{R} GPUs, {args.groups} groups, {args.per_rank_mib} MiB/rank ratio {args.ratio} hot rank {args.hot}: "
          f"mismatched {bad}", flush=True)


if __name__ == "__main__":
    main()
