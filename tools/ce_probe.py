"""What would copy engines reach on the BASELINE all-to-allv patterns?

One process drives every GPU of the box.  Each rank's segments are sent with
cudaMemcpyAsync peer copies (cuda-python runtime calls, peer access on: the
copy engines move the bytes, no SM involved), one stream per (sender,
receiver) pair so a sender's copies run concurrently, or one per sender.  Timed with events on
each sender's streams after a device-wide start; per call the max over
GPUs; median of `iters`.  Reports the fraction of the MCF port bound
(900 GB/s per port) beside the same matrix's bound -- the ceiling a copy
engine data path would have, against the SM engine's measured fraction.

  python tools/ce_probe.py [per_rank_mib]      (prints one JSON line per case)
"""
import json
import os
import sys
import time

import torch
from cuda.bindings import runtime as cudart

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def port_bound(m, R):
    return max(max(sum(m[v * R + d] for d in range(R) if d != v), sum(m[s * R + v] for s in range(R) if s != v))
               for v in range(R)) / 900e9


def run_case(R, m, iters=20, warmup=3, per_pair_stream=True):
    sends, recvs = [], []
    for r in range(R):
        with torch.cuda.device(r):
            sends.append(torch.empty(max(sum(m[r * R + d] for d in range(R)), 16), dtype=torch.uint8, device=r))
            recvs.append(torch.empty(max(sum(m[s * R + r] for s in range(R)), 16), dtype=torch.uint8, device=r))
    soff = [[sum(m[s * R + x] for x in range(d)) for d in range(R)] for s in range(R)]
    roff = [[sum(m[x * R + d] for x in range(s)) for s in range(R)] for d in range(R)]
    streams = {}
    for s in range(R):
        for d in range(R):
            if s != d and m[s * R + d]:
                key = (s, d) if per_pair_stream else (s, 0)
                if key not in streams:
                    streams[key] = torch.cuda.Stream(device=s)
    for r in range(R):
        torch.cuda.synchronize(r)

    def one():
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        for s in range(R):
            starts[s].record(torch.cuda.current_stream(s))
        ends = []
        for s in range(R):
            for d in range(R):
                n = m[s * R + d]
                if s == d or not n:
                    continue
                st = streams[(s, d) if per_pair_stream else (s, 0)]
                st.wait_event(starts[s])
                err, = cudart.cudaMemcpyAsync(recvs[d].data_ptr() + roff[d][s], sends[s].data_ptr() + soff[s][d], n,
                                              cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice, st.cuda_stream)
                assert err == cudart.cudaError_t.cudaSuccess, err
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                ends.append((s, e))
        for r in range(R):
            torch.cuda.synchronize(r)
        return max(starts[s].elapsed_time(e) for s, e in ends) * 1e-3

    for _ in range(warmup):
        one()
    ts = sorted(one() for _ in range(iters))
    t = ts[len(ts) // 2]
    b = port_bound(m, R)
    return {"us": t * 1e6, "bound_us": b * 1e6, "frac_of_bound": b / t, "gbps": sum(m) / t / 1e9}


def enable_peers(R):
    for a in range(R):
        cudart.cudaSetDevice(a)
        for b in range(R):
            if a != b:
                err, = cudart.cudaDeviceEnablePeerAccess(b, 0)
                assert err in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
    cudart.cudaSetDevice(0)


def main():
    R = torch.cuda.device_count()
    for r in range(R):
        torch.zeros(1, device=r)  # contexts first
    enable_peers(R)
    per_rank = int(sys.argv[1]) * MiB if len(sys.argv) > 1 else 256 * MiB
    cases = [("c5", P.gen_skewed_a2av(R, per_rank, 1.0 / (R - 1), 0), {})]
    for r in (0.0, 0.3, 0.5, 0.7, 0.9):
        cases.append(("c3", P.gen_skewed_a2av(R, per_rank, r, 0), {"ratio": r}))
    cases.append(("p2p", P.gen_p2p(R, 0, 1, per_rank), {}))
    for name, m, extra in cases:
        for pps in (True, False):
            res = run_case(R, m, per_pair_stream=pps)
            print(json.dumps(dict(case=name, ranks=R, per_rank=per_rank, engine="copy engine",
                                  streams="per pair" if pps else "per sender", **extra, **res)), flush=True)


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(f"# {time.time() - t0:.1f} s", file=sys.stderr)
