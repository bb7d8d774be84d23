"""Quick GPU probe (development aid): local emulated exchange, then, under
torchrun, the multi-process data path.  Prints one line per check."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def local_probe(per_rank, ratio, iters=10, ctas=0):
    R = 8
    m = P.gen_skewed_a2av(R, per_rank, ratio, 0)
    sends, recvs = [], []
    for s in range(R):
        row = sum(m[s * R:(s + 1) * R])
        col = sum(m[x * R + s] for x in range(R))
        sends.append(torch.empty(max(row, 16), dtype=torch.uint8, device="cuda"))
        recvs.append(torch.zeros(max(col, 16), dtype=torch.uint8, device="cuda"))
    for s in range(R):
        sc, sd, rc, rd = C.packed_displs(m, R, s)
        for d in range(R):
            C.fill_payload(sends[s][sd[d]:], 0, sc[d], 1, s, d)
    C.exchange_local(sends, recvs, m, ctas)
    torch.cuda.synchronize()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for d in range(R):
        sc, sd, rc, rd = C.packed_displs(m, R, d)
        for s in range(R):
            C.check_payload(recvs[d][rd[s]:], 0, rc[s], 1, s, d, bad)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        C.exchange_local(sends, recvs, m, ctas)
    ts = []
    for _ in range(iters):
        ev[0].record()
        C.exchange_local(sends, recvs, m, ctas)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e-3)
    ts.sort()
    t = ts[len(ts) // 2]
    total = sum(m)
    print(f"local R=8 per_rank={per_rank>>20}MiB r={ratio} ctas={ctas}: mismatches={int(bad.item())} "
          f"t={t*1e3:.3f}ms eff={total/t/1e9:.1f}GB/s hbm(r+w)={2*total/t/1e9:.1f}GB/s", flush=True)


def mp_probe():
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    obj = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, 0)
    t0 = time.time()
    comm = C.Comm.init_rank(world, obj[0], rank)
    if rank == 0:
        print(f"comm init {time.time()-t0:.2f}s", flush=True)
    for ratio in (0.0, 0.7):
        r = comm.bench_skewed(64 * MiB, ratio, 0, warmup=2, iters=5)
        if rank == 0:
            print(f"bench_skewed R={world} 64MiB r={ratio}: {r}", flush=True)
    r = comm.bench_p2p(64 * MiB, 0, 1, warmup=2, iters=5)
    if rank == 0:
        print(f"bench_p2p 64MiB: {r}", flush=True)
    # staged (unregistered receive) path
    R = world
    m = P.gen_skewed_a2av(R, 8 * MiB + 13, 0.7, 0)
    sc, sd, rc, rd = C.packed_displs(m, R, rank)
    send = torch.empty(sum(sc) + 16, dtype=torch.uint8, device="cuda")
    recv = torch.zeros(sum(rc) + 16, dtype=torch.uint8, device="cuda")
    for d in range(R):
        C.fill_payload(send[sd[d]:], 0, sc[d], 7, rank, d)
    comm.alltoallv(send, sc, sd, recv, rc, rd)
    torch.cuda.synchronize()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s in range(R):
        C.check_payload(recv[rd[s]:], 0, rc[s], 7, s, rank, bad)
    torch.cuda.synchronize()
    comm.check_async()
    print(f"rank {rank} staged alltoallv mismatches={int(bad.item())}", flush=True)
    # relay path (mesh model)
    comm.set_config(fabric="alltoall", gpus_per_node=R)
    r = comm.bench_p2p(256 * MiB, 0, 1, warmup=1, iters=3)
    if rank == 0:
        print(f"relay bench_p2p 256MiB mesh{R}: {r}", flush=True)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        mp_probe()
    else:
        local_probe(8 * MiB + 5, 0.7, iters=3)
        for ctas in (0, 74, 296):
            local_probe(256 * MiB, 0.7, ctas=ctas)
