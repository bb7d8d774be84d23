"""Device timeline of one exchange on every rank (development aid; torchrun, NIMBLE_TRACE=1)."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20
NAMES = ["start", "prolog", "first", "last", "ctas", "signal", "waited", "cta0done", "loopsmax", "fencemax", "loopsmin",
         "entry", "prevend"]


def _pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * (len(v) - 1) + 0.5))] if v else float("nan")


def cta_summary(t0, ctas):
    """Per-CTA timeline: quantiles (min / median / max, us from kernel
    start) of queue-empty, loops-done and fence-done, and the fence's
    duration for CTAs that stored into peers vs those that did not."""
    us = lambda x: (x - t0) / 1e3  # noqa: E731
    out = [f"{len(ctas)} CTAs ({sum(1 for c in ctas if c[4])} with peer stores)"]
    for name, k in (("first", 0), ("qempty", 1), ("loops", 2), ("fence", 3)):
        v = [us(c[k]) for c in ctas if c[k]]
        out.append(f"{name} {_pct(v, 0):.1f}/{_pct(v, .5):.1f}/{_pct(v, 1):.1f}")
    for tag, sel in (("remote", lambda c: c[4] > 0), ("local", lambda c: c[4] == 0)):
        d = [(c[3] - c[2]) / 1e3 for c in ctas if sel(c) and c[3] and c[2]]
        if d:
            out.append(f"fence[{tag}] {_pct(d, 0):.1f}/{_pct(d, .5):.1f}/{_pct(d, 1):.1f}")
    mb = [(c[4] + c[5]) / 2**20 for c in ctas]
    out.append(f"MiB/CTA {_pct(mb, 0):.2f}/{_pct(mb, .5):.2f}/{_pct(mb, 1):.2f}")
    return "  ".join(out)


def main():
    os.environ["NIMBLE_TRACE"] = "1"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    uid = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    comm = C.Comm.init_rank(world, uid[0], rank)
    R = world
    case = os.environ.get("TRACE_CASE", "skew")
    if case == "relay":
        comm.set_config(fabric="alltoall", gpus_per_node=R)
    for pull in [int(v) for v in os.environ.get("TRACE_PULL", "1,2").split(",")]:
        comm.set_config(pull=pull)
        sizes = [int(v) for v in os.environ.get("TRACE_KIB", "65536,1048576" if case == "relay" else "1024,262144").split(",")]
        for kib in sizes:
            mib = kib / 1024
            if case == "relay":
                m = P.gen_p2p(R, 0, 1, kib * 1024)
            elif case == "irregular":  # c4: total bytes over the whole matrix
                m = P.gen_irregular(R, kib * 1024, 0.5, 1)
            else:
                m = P.gen_skewed_a2av(R, kib * 1024, float(os.environ.get("TRACE_RATIO", "0.7")), 0)
            sc, sd, rc, rd = C.packed_displs(m, R, rank)
            send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
            recv = torch.empty(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
            hs, hr = comm.register(send), comm.register(recv)
            for _ in range(5):
                comm.alltoallv(send, sc, sd, recv, rc, rd)
            tr = comm.debug_trace(per_cta=True)
            allt = [None] * world
            dist.all_gather_object(allt, tr)
            if rank == 0:
                print(f"pull={pull} {kib} KiB/rank (us from each rank's own kernel start; globaltimers differ across GPUs)")
                for r, (t, ctas) in enumerate(allt):
                    print(f"  rank {r}: " + " ".join(f"{n}={(v - t[0]) / 1e3:6.1f}" for n, v in zip(NAMES, t[:13])),
                          flush=True)
                    print("    " + cta_summary(t[0], ctas), flush=True)
            comm.deregister(hs)
            comm.deregister(hr)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
