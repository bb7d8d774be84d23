"""Per-call cost of exchanges whose counts change every call (MoE-style).

Each rank runs K alltoallv calls, each with a new count matrix (seeded,
identical on every rank): plan + schedule (device-generated) + launch per
call.  Reports the host microseconds per call (the C ABI call, measured
around it) and the device time per call, beside the same numbers for a
matrix repeated every call (cached schedule).

  co-resident on one GPU:   python tools/fresh_matrix_probe.py --threads 8
  one process per GPU:      torchrun --nproc-per-node N tools/fresh_matrix_probe.py
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import torch

os.environ.setdefault("NIMBLE_STATS", "1")  # the comm's host / device counters
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import fresh_matrices  # noqa: E402
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def run_rank(comm, rank, R, args, barrier):
    base = P.gen_skewed_a2av(R, args.per_rank_mib * MiB, args.ratio, 0)
    mats = fresh_matrices(base, R, args.calls + 8, seed=99)
    sc, sd, rc, rd = C.packed_displs(base, R, rank)
    send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
    recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
    hs = [comm.register(send), comm.register(recv)]
    st = torch.cuda.current_stream()
    out = {}
    for mode in ("repeat", "fresh"):
        lays = [C.packed_displs(mats[k] if mode == "fresh" else base, R, rank) for k in range(args.calls + 8)]
        for k in range(8):  # warm-up (distinct matrices too)
            a, b, c, d = lays[args.calls + k]
            comm.alltoallv(send, a, b, recv, c, d)
        st.synchronize()
        comm.stats(reset=True)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        host = []
        e0.record()
        for k in range(args.calls):
            a, b, c, d = lays[k]
            t0 = time.perf_counter()
            comm.alltoallv(send, a, b, recv, c, d)
            host.append(time.perf_counter() - t0)
        e1.record()
        st.synchronize()
        cs = comm.stats()
        out[mode] = {"python_us_median": statistics.median(host) * 1e6,
                     "c_abi_us_mean": cs["host_ns"] / max(cs["host_calls"], 1) / 1e3,
                     "c_abi_us_max": cs["host_ns_max"] / 1e3,
                     "plans_built": cs["plans_built"], "plan_us_mean": cs["plan_ns"] / max(cs["plans_built"], 1) / 1e3,
                     "schedules_built": cs["schedules_built"],
                     "schedule_us_mean": cs["schedule_ns"] / max(cs["schedules_built"], 1) / 1e3,
                     "device_ms_per_call": e0.elapsed_time(e1) / args.calls}
        barrier()
    comm.check_async()
    for h in hs:
        comm.deregister(h)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0, help="R co-resident ranks on GPU 0 (0: torchrun layout)")
    ap.add_argument("--per-rank-mib", type=int, default=256)
    ap.add_argument("--ratio", type=float, default=0.7)
    ap.add_argument("--calls", type=int, default=30)
    args = ap.parse_args()
    if args.threads:
        R = args.threads
        uid = C.unique_id()
        bar = threading.Barrier(R)
        res = [None] * R

        def th(r):
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                comm = C.Comm.init_rank(R, uid, r)
                res[r] = run_rank(comm, r, R, args, lambda: bar.wait())
                s.synchronize()
                bar.wait()
                comm.destroy()

        ts = [threading.Thread(target=th, args=(r,)) for r in range(R)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        print(json.dumps({"layout": f"{R} ranks co-resident on 1 GPU", "per_rank_mib": args.per_rank_mib,
                          "ratio": args.ratio, "ranks": res}))
        return
    import torch.distributed as dist
    rank, R = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    uid = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    comm = C.Comm.init_rank(R, uid[0], rank)
    r = run_rank(comm, rank, R, args, dist.barrier)
    allr = [None] * R
    dist.all_gather_object(allr, r)
    if rank == 0:
        print(json.dumps({"layout": f"{R} ranks, 1 per GPU", "per_rank_mib": args.per_rank_mib, "ratio": args.ratio,
                          "ranks": allr}))
    comm.destroy()


if __name__ == "__main__":
    main()
