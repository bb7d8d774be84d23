"""MoE dispatch + combine throughput: nimble vs NCCL (torchrun, one process per GPU).

DeepSeek-like shapes (H = 7168 bf16, top-8 of 64 experts), T tokens per rank,
router skewed towards experts on rank 0 with probability MOE_HOT.  Both arms
do identical index bookkeeping; only the exchanges differ (nimble
alltoallv vs torch.distributed.all_to_all_single on NCCL).  Prints one JSON
line per hot probability on rank 0.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200.moe import MoEDispatcher  # noqa: E402


def nccl_dispatch_combine(pg, x, ids, epr, R, w):
    T, k = ids.shape
    flat = ids.reshape(-1)
    dest = flat // epr
    order = torch.argsort(dest, stable=True)
    send = x.index_select(0, order // k)
    cnt = torch.bincount(dest, minlength=R)
    rcnt = torch.empty_like(cnt)
    dist.all_to_all_single(rcnt, cnt, group=pg)
    sc, rc = cnt.tolist(), rcnt.tolist()
    recv = torch.empty(sum(rc), x.shape[1], dtype=x.dtype, device=x.device)
    dist.all_to_all_single(recv, send, rc, sc, group=pg)
    back = torch.empty_like(send)
    dist.all_to_all_single(back, recv, sc, rc, group=pg)
    out = torch.zeros_like(x)
    out.index_add_(0, order // k, back * w.reshape(-1)[order].to(x.dtype).unsqueeze(1))
    return out, sum(rc)


def main():
    os.environ["NCCL_DEBUG"] = "WARN"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    pg = dist.new_group(backend="nccl")
    uid = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    comm = C.Comm.init_rank(world, uid[0], rank)
    T, H, k, E = int(os.environ.get("MOE_T", "4096")), 7168, 8, 64
    disp = MoEDispatcher(comm, E, H, dtype=torch.bfloat16, max_tokens=T, topk=k)
    g = torch.Generator(device="cuda").manual_seed(rank)
    x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16, generator=g)
    w = torch.rand(T, k, device="cuda", generator=g)
    for hot in [float(v) for v in os.environ.get("MOE_HOT", "0.0,0.5,0.8").split(",")]:
        # hot assignments go to rank 0's experts; the rest are uniform
        is_hot = torch.rand(T, k, device="cuda", generator=g) < hot
        ids = torch.where(is_hot, torch.randint(0, disp.experts_per_rank, (T, k), device="cuda", generator=g),
                          torch.randint(0, E, (T, k), device="cuda", generator=g))

        def nimble_step():
            rx, re, h = disp.dispatch(x, ids)
            return disp.combine(rx, h, w), sum(h.recv_counts)

        res = {}
        for name, fn in (("nimble", nimble_step), ("nccl", lambda: nccl_dispatch_combine(
                pg, x, ids, disp.experts_per_rank, world, w))):
            for _ in range(3):
                out, rows = fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            n = 10
            for _ in range(n):
                out, rows = fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / n], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[name] = (float(t.item()), out)
        same = torch.allclose(res["nimble"][1].float(), res["nccl"][1].float(), rtol=2e-2, atol=2e-2)
        # the row exchanges alone (dispatch direction), same buffers and counts for both arms
        rx, re, h = disp.dispatch(x, ids)
        sb = [c * disp.row for c in h.send_counts]
        rb = [c * disp.row for c in h.recv_counts]
        sd, rd = disp._displs(sb), disp._displs(rb)
        def ex_nimble():
            comm.alltoallv(disp.send_buf, sb, sd, disp.recv_buf, rb, rd)
        sv = disp.send_buf[:sum(h.send_counts)]
        rv = disp.recv_buf[:sum(h.recv_counts)]
        def ex_nccl():
            dist.all_to_all_single(rv, sv, list(h.recv_counts), list(h.send_counts), group=pg)
        ex = {}
        for name, fn in (("nimble", ex_nimble), ("nccl", ex_nccl)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(10):
                fn()
            a1.record()
            torch.cuda.synchronize()
            tt = torch.tensor([a0.elapsed_time(a1) * 1e-3 / 10], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ex[name] = float(tt.item())
        bytes_moved = torch.tensor([T * k * H * 2 * 2], dtype=torch.float64)  # dispatch + combine, this rank
        dist.all_reduce(bytes_moved)
        if rank == 0:
            print(json.dumps({"world": world, "tokens_per_rank": T, "hidden": H, "topk": k, "experts": E,
                              "hot_prob": hot, "nimble_ms": res["nimble"][0] * 1e3, "nccl_ms": res["nccl"][0] * 1e3,
                              "nimble_tokens_per_s": T * world / res["nimble"][0],
                              "nccl_tokens_per_s": T * world / res["nccl"][0],
                              "speedup": res["nccl"][0] / res["nimble"][0],
                              "payload_gbps_nimble": float(bytes_moved.item()) / res["nimble"][0] / 1e9,
                              "dispatch_exchange_ms": {k2: v * 1e3 for k2, v in ex.items()},
                              "outputs_match": bool(same)}), flush=True)
    disp.close()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
