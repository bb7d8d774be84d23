"""BASELINE.json config sweeps on real GPUs (torchrun, one process per GPU).

For the world size it is launched with (W), rank 0 prints one JSON line per
point: nimble GB/s, fraction of the MCF port bound, NCCL all_to_all_single on
the same buffers, relay flows, delivery mismatches.  Times: 5 warm-up + 100
timed rounds (SWEEP_ITERS), per-round CUDA events, max over ranks per round;
`us` is the median, `us_min` / `us_mean` beside it; `us_block` times the same
calls back to back between two events (bench.py's protocol, where
consecutive exchanges chain without an event between them).
  c3  skewed all-to-allv, 256 MiB/rank, hotspot ratio 0.0 .. 0.9
  c5  uniform all-to-allv (ratio 1/(W-1)), 256 MiB/rank
  c4  irregular seeded matrix (seed 1, sparsity 0.5), total 1 KiB .. 1 GiB
  c1  p2p 64 MiB 0 -> 1 (W = 3: one relay GPU under the mesh model)
  c2  p2p 1 GiB 0 -> 1 (W = 4: two relay GPUs under the mesh model)
  cal p2p 256 MiB 0 -> 1, direct and through W - 2 relays (calibration targets)
SWEEP_CASES selects (default all that fit W).
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import comm as C  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def max_over(x):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def port_bound(m, R):
    return max(max(sum(m[v * R + d] for d in range(R) if d != v), sum(m[s * R + v] for s in range(R) if s != v))
               for v in range(R)) / 900e9


def timed(fn, st, iters, warmup):
    """Per-iteration device times (CUDA events on `st`), max over ranks per
    iteration; returns (median, min, mean) seconds.  Protocol of the
    reference's bench (5 warm-up + 100 timed rounds)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
    ev[0].record(st)
    for i in range(iters):
        fn()
        ev[i + 1].record(st)
    torch.cuda.synchronize()
    per = torch.tensor([ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(iters)], dtype=torch.float64)
    dist.all_reduce(per, op=dist.ReduceOp.MAX)
    v = sorted(per.tolist())
    return v[len(v) // 2], v[0], sum(v) / len(v)


def nvml_read():
    """NVLink byte counters of this rank's GPU (SWEEP_NVML=1), else None."""
    if os.environ.get("SWEEP_NVML") != "1":
        return None
    try:
        from tools import nvml_nvlink
        return nvml_nvlink.read(torch.cuda.current_device())
    except Exception as e:  # driver without the counters
        return {"error": str(e)[:80]}


def nvml_delta(a, b, calls):
    if a is None or b is None or "error" in a or "error" in b:
        return a if a and "error" in a else None
    return {k: (b[k] - a[k]) / calls if a[k] is not None and b[k] is not None else None for k in a}


def timed_graph(fn, st, iters, warmup):
    """`iters` calls captured in one CUDA graph, replayed once: per-call device
    time without host launch overhead (max over ranks).  Returns seconds."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(iters):
            fn()
    g.replay()  # warm replay
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    return max_over(e0.elapsed_time(e1) * 1e-3 / iters)


def timed_block(fn, st, iters, warmup):
    """`iters` back-to-back calls between two events (bench.py's protocol: no
    event between calls, so consecutive exchanges chain), per-call mean, max
    over ranks.  Returns seconds."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return max_over(e0.elapsed_time(e1) * 1e-3 / iters)


def _run_point(comm, pg, rank, R, m, name, fabric="nvswitch", iters=None, warmup=5, nccl=True, extra=None):
    iters = iters or int(os.environ.get("SWEEP_ITERS", "100"))
    comm.set_config(fabric=fabric, gpus_per_node=R)
    sc, sd, rc, rd = C.packed_displs(m, R, rank)
    send = torch.empty(max(sum(sc), 16), dtype=torch.uint8, device="cuda")
    recv = torch.zeros(max(sum(rc), 16), dtype=torch.uint8, device="cuda")
    for d in range(R):
        C.fill_payload(send[sd[d]:], 0, sc[d], 9, rank, d)
    hs, hr = comm.register(send), comm.register(recv)
    st = torch.cuda.current_stream()
    nvl0 = nvml_read()
    t, t_min, t_mean = timed(lambda: comm.alltoallv(send, sc, sd, recv, rc, rd, st), st, iters, warmup)
    nvl = nvml_delta(nvl0, nvml_read(), iters + warmup)
    tb = timed_block(lambda: comm.alltoallv(send, sc, sd, recv, rc, rd, st), st, iters, warmup)
    comm.check_async()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s in range(R):
        C.check_payload(recv[rd[s]:], 0, rc[s], 9, s, rank, bad)
    torch.cuda.synchronize()
    mism = int(max_over(float(bad.item())))
    tn = None
    if nccl:
        out = torch.empty_like(recv)
        sv, rv = send[:sum(sc)], out[:sum(rc)]
        tn, _, _ = timed(lambda: dist.all_to_all_single(rv, sv, list(rc), list(sc), group=pg), st, iters, warmup)
        tnb = timed_block(lambda: dist.all_to_all_single(rv, sv, list(rc), list(sc), group=pg), st, iters, warmup)
    graph = None
    if os.environ.get("SWEEP_GRAPH") == "1":  # host overhead removed, both arms
        st2 = torch.cuda.Stream()
        with torch.cuda.stream(st2):
            graph = {"nimble_us": timed_graph(lambda: comm.alltoallv(send, sc, sd, recv, rc, rd, st2), st2, iters,
                                              warmup) * 1e6}
            if nccl:
                graph["nccl_us"] = timed_graph(lambda: dist.all_to_all_single(rv, sv, list(rc), list(sc), group=pg),
                                               st2, iters, warmup) * 1e6
    comm.deregister(hs)
    comm.deregister(hr)
    total = sum(m)
    bound = port_bound(m, R)
    relays = 0
    if fabric == "alltoall":
        t_ = P.build_canonical(1, R, 0, 900e9, 0, P.ALLTOALL)
        relays = sum(1 for pp in P.plan(t_, R, R, m).pairs for c, _ in pp.flows if c > 0)
    row = {"case": name, "ranks": R, "fabric_model": fabric, "total_bytes": total, "us": t * 1e6,
           "us_min": t_min * 1e6, "us_mean": t_mean * 1e6, "iters": iters, "warmup": warmup,
           "gbps": total / t / 1e9, "bound_us": bound * 1e6, "frac_of_bound": bound / t if t else None,
           "nccl_us": tn * 1e6 if tn else None, "nccl_gbps": total / tn / 1e9 if tn else None,
           "vs_nccl": (tn / t) if tn else None, "relay_flows": relays, "mismatched_bytes": mism,
           # back-to-back calls between two events (bench.py's protocol)
           "us_block": tb * 1e6, "frac_of_bound_block": bound / tb if tb else None,
           "nccl_us_block": tnb * 1e6 if tn else None, "vs_nccl_block": (tnb / tb) if tn else None}
    if graph:
        row["graph"] = graph
    if nvl is not None:  # this rank's NVLink counters per call (rank 0 prints its own; hot rank = 0)
        row["nvlink_per_call_rank0"] = nvl
        sent = sum(m[rank * R + d] for d in range(R) if d != rank)
        got = sum(m[s * R + rank] for s in range(R) if s != rank)
        row["payload_per_call_rank0"] = {"egress": sent, "ingress": got}
    if extra:
        row.update(extra)
    if rank == 0:
        print(json.dumps(row), flush=True)
    return row


def main():
    os.environ["NCCL_DEBUG"] = "WARN"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    pg = dist.new_group(backend="nccl")
    uid = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    comm = C.Comm.init_rank(world, uid[0], rank)
    if os.environ.get("SWEEP_PULL"):
        comm.set_config(pull=int(os.environ["SWEEP_PULL"]))
    if os.environ.get("SWEEP_LL_MAX"):
        comm.set_config(ll_max=int(os.environ["SWEEP_LL_MAX"]))
    if os.environ.get("SWEEP_PUSH_CHUNK"):
        comm.set_config(push_chunk=int(os.environ["SWEEP_PUSH_CHUNK"]))
    if os.environ.get("SWEEP_CTAS"):
        comm.set_config(ctas=int(os.environ["SWEEP_CTAS"]))
    if os.environ.get("SWEEP_PIPE_CHUNK"):  # relay staging geometry (pipe_chunk, p2p_buffer)
        comm.set_config(pipe_chunk=int(os.environ["SWEEP_PIPE_CHUNK"]),
                        p2p_buffer=int(os.environ.get("SWEEP_P2P_BUFFER", str(10 << 20))))
    for chunk in [int(v) for v in os.environ.get("SWEEP_CHUNKS", "0").split(",")]:
        comm.set_config(direct_chunk=chunk)
        sweep(comm, pg, rank, world, chunk)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def sweep(comm, pg, rank, world, chunk):
    R = world
    cases = os.environ.get("SWEEP_CASES", "c3,c5,c4,c1,c2").split(",")
    per_rank = int(os.environ.get("SWEEP_PER_RANK_MIB", "256")) * MiB
    nccl = os.environ.get("SWEEP_NCCL", "1") == "1"
    tag = {"direct_chunk": chunk} if chunk else {}

    def run_point(*a, extra=None, **k):
        return _run_point(*a, nccl=nccl, extra=dict(extra or {}, **tag), **k)
    if "c3" in cases:
        for i in range(10):
            run_point(comm, pg, rank, R, P.gen_skewed_a2av(R, per_rank, i / 10, 0), "c3",
                      extra={"ratio": i / 10, "per_rank": per_rank})
    if "c3a" in cases:  # the same skew with every pair rounded down to 256 B (NCCL's aligned fast path)
        for i in (0, 3, 5, 7, 9):
            m = [v // 256 * 256 for v in P.gen_skewed_a2av(R, per_rank, i / 10, 0)]
            run_point(comm, pg, rank, R, m, "c3a", extra={"ratio": i / 10, "per_rank": per_rank})
    if "c5" in cases:
        run_point(comm, pg, rank, R, P.gen_skewed_a2av(R, 256 * MiB, 1.0 / (R - 1), 0), "c5")
    if "c3k" in cases:  # small skewed exchanges: 64 KiB .. 4 MiB per rank, r = 0.7
        for kib in (64, 256, 1024, 4096):
            run_point(comm, pg, rank, R, P.gen_skewed_a2av(R, kib << 10, 0.7, 0), "c3k",
                      extra={"ratio": 0.7, "per_rank": kib << 10})
    if "c4" in cases:
        t = 1024
        while t <= 1 << 30:
            run_point(comm, pg, rank, R, P.gen_irregular(R, t, 0.5, 1), "c4", extra={"total": t})
            t *= 16
    if "cal" in cases and R >= 3:  # calibration points: p2p 256 MiB direct vs R-2 relays (mesh plan)
        for fab in ("nvswitch", "alltoall"):
            run_point(comm, pg, rank, R, P.gen_p2p(R, 0, 1, 256 * MiB), "cal", fab, extra={"per_rank": 256 * MiB})
    if "c1" in cases and R == 3:
        for fab in ("nvswitch", "alltoall"):
            run_point(comm, pg, rank, R, P.gen_p2p(R, 0, 1, 64 * MiB), "c1", fab)
    if "c2" in cases and R == 4:
        for fab in ("nvswitch", "alltoall"):
            run_point(comm, pg, rank, R, P.gen_p2p(R, 0, 1, 1 << 30), "c2", fab, iters=20)


if __name__ == "__main__":
    main()
