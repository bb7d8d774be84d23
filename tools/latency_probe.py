"""Per-call host cost and back-to-back device latency (development aid; torchrun)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    uid = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    comm = C.Comm.init_rank(world, uid[0], rank)
    R = world
    pulls = [int(v) for v in os.environ.get("LAT_PULL", "1,2").split(",")]
    chunks = [int(v) for v in os.environ.get("LAT_CHUNKS", "0").split(",")]
    sizes = [int(v) for v in os.environ.get("LAT_KIB", "1024,16384,262144").split(",")]
    for pull, chunk in [(p, c) for p in pulls for c in chunks]:
        comm.set_config(pull=pull, direct_chunk=chunk)
        for kib in sizes:
            m = P.gen_skewed_a2av(R, kib * 1024, 0.7, 0)
            sc, sd, rc, rd = C.packed_displs(m, R, rank)
            send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
            recv = torch.empty(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
            hs, hr = comm.register(send), comm.register(recv)
            st = torch.cuda.current_stream()
            for _ in range(5):
                comm.alltoallv(send, sc, sd, recv, rc, rd, st)
            torch.cuda.synchronize()
            dist.barrier()
            n = 50
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(st)
            for _ in range(n):
                comm.alltoallv(send, sc, sd, recv, rc, rd, st)
            e1.record(st)
            host = (time.perf_counter() - t0) / n
            torch.cuda.synchronize()
            dev = e0.elapsed_time(e1) * 1e-3 / n
            t = torch.tensor([dev, host], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            comm.check_async()
            if rank == 0:
                bound = max(sum(m[s * R + v] for s in range(R) if s != v) for v in range(R)) / 900e9
                print(f"pull={pull} chunk={chunk:6d} {kib:7d}KiB: device {t[0]*1e6:8.1f}us/call  host {t[1]*1e6:6.1f}us/call "
                      f"bound {bound*1e6:7.1f}us frac {bound/t[0]:.3f}", flush=True)
            comm.deregister(hs)
            comm.deregister(hr)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
