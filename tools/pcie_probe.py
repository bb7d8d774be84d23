"""PCIe host<->device bandwidth on one GPU: the ceiling of bench.py's e2e leg.

Measures pinned H2D alone, D2H alone, both at once (full duplex), with and
without binding the process to the GPU's local CPUs / NUMA node first, and
for a few copy sizes.  One JSON line per measurement.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

GiB = 1 << 30


def local_cpus(dev=0):
    import subprocess
    bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                         capture_output=True, text=True).stdout.strip().lower()
    if bus.startswith("0000") and len(bus.split(":")[0]) == 8:
        bus = bus[4:]
    for cand in (bus, "0000" + bus[4:] if bus.startswith("00000000") else bus):
        p = f"/sys/bus/pci/devices/{cand}/local_cpulist"
        if os.path.exists(p):
            s = open(p).read().strip()
            cpus = set()
            for part in s.split(","):
                a, _, b = part.partition("-")
                cpus.update(range(int(a), int(b or a) + 1))
            node = open(f"/sys/bus/pci/devices/{cand}/numa_node").read().strip()
            return cpus, node, cand
    return None, None, bus


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / iters


def run(tag, nbytes, chunks=1):
    h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_in.fill_(1)
    h_out.fill_(2)
    d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cs = nbytes // chunks

    def h2d():
        for i in range(chunks):
            d_in[i * cs:(i + 1) * cs].copy_(h_in[i * cs:(i + 1) * cs], non_blocking=True)

    def d2h():
        for i in range(chunks):
            h_out[i * cs:(i + 1) * cs].copy_(d_out[i * cs:(i + 1) * cs], non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            h2d()
        with torch.cuda.stream(s2):
            d2h()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    r = {"tag": tag, "bytes": nbytes, "chunks": chunks,
         "h2d_gbs": nbytes / timed(h2d) / 1e9, "d2h_gbs": nbytes / timed(d2h) / 1e9}
    tb = timed(both)
    r["duplex_gbs_each"] = nbytes / tb / 1e9
    print(json.dumps(r), flush=True)
    del h_in, h_out, d_in, d_out


def main():
    torch.cuda.set_device(0)
    cpus, node, bus = local_cpus(0)
    print(json.dumps({"bus": bus, "numa_node": node, "local_cpus": len(cpus) if cpus else None,
                      "affinity_before": len(os.sched_getaffinity(0)), "cpu_count": os.cpu_count()}), flush=True)
    run("default", GiB)
    run("default", 256 << 20)
    run("default-chunked16", GiB, 16)
    if cpus:
        allowed = cpus & os.sched_getaffinity(0)
        if allowed:
            os.sched_setaffinity(0, allowed)
            run("numa-local", GiB)
            run("numa-local", 2 * GiB)
            run("numa-local-chunked16", GiB, 16)


if __name__ == "__main__":
    main()
