"""Regenerate the golden fixtures in tests/golden/ from the compiled reference.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_golden.py

Every fixture is the reference's own output (oracle/_ref/libnimble_ref.so, the
unmodified proj/src/*.cpp) for a request that is stored next to it, so tests
can replay the request against the Python oracle and against the product's
C-ABI without /root/reference being present.
"""
from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

MiB = 1 << 20
KiB = 1 << 10
GiB = 1 << 30


def topo(gpus, fabric, nodes=1, nics=0, nvlink=900.0, rail=50.0):
    return {"nodes": nodes, "gpus": gpus, "nics": nics, "fabric": fabric,
            "nvlink_gbps": nvlink, "rail_gbps": rail}


def config_requests():
    """The BASELINE.json configs c1..c5."""
    out = []
    # c1: p2p 64 MiB, 2 ranks, direct + 1 relay (alltoall g=3) and nvswitch g=2
    out.append(("c1_mesh3", {"ranks": 2, "ranks_per_node": 3, "topology": topo(3, "alltoall"),
                             "workload": {"kind": "p2p", "size": 64 * MiB}}))
    out.append(("c1_nvswitch2", {"ranks": 2, "topology": topo(2, "nvswitch"),
                                 "workload": {"kind": "p2p", "size": 64 * MiB}}))
    # c2: p2p 1 GiB, 2 relays (alltoall g=4) and nvswitch g=8
    out.append(("c2_mesh4", {"ranks": 2, "ranks_per_node": 4, "topology": topo(4, "alltoall"),
                             "workload": {"kind": "p2p", "size": GiB}}))
    out.append(("c2_nvswitch8", {"ranks": 2, "ranks_per_node": 8, "topology": topo(8, "nvswitch"),
                                 "workload": {"kind": "p2p", "size": GiB}}))
    # c3: skewed all-to-allv, 8 GPUs, 256 MiB/rank (and 64 MiB/rank), ratio sweep
    for per in (64 * MiB, 256 * MiB):
        for i in range(10):
            r = i / 10
            out.append((f"c3_nvswitch8_{per // MiB}m_r{i}",
                        {"ranks": 8, "topology": topo(8, "nvswitch"),
                         "workload": {"kind": "skewed", "size": per, "ratio": r, "hot": 0}}))
    for i in (5, 7, 9):
        out.append((f"c3_mesh8_256m_r{i}",
                    {"ranks": 8, "topology": topo(8, "alltoall"),
                     "workload": {"kind": "skewed", "size": 256 * MiB, "ratio": i / 10, "hot": 0}}))
    # c4: irregular seeded, 8 GPUs, 1 KiB .. 1 GiB in 4x steps
    t = KiB
    while t <= GiB:
        out.append((f"c4_nvswitch8_{t}", {"ranks": 8, "topology": topo(8, "nvswitch"),
                                          "workload": {"kind": "irregular", "size": t,
                                                       "sparsity": 0.5, "seed": 1}}))
        t *= 4
    # c5: uniform all-to-allv (skewed at ratio 1/(R-1)), R = 2, 4, 8
    for R in (2, 4, 8):
        out.append((f"c5_nvswitch{R}", {"ranks": R, "topology": topo(R, "nvswitch"),
                                        "workload": {"kind": "skewed", "size": 256 * MiB,
                                                     "ratio": 1.0 / (R - 1), "hot": 0}}))
    return out


def fuzz_requests(n, seed):
    """Random planner instances in the style of acceptance.cpp:304-389."""
    rng = random.Random(seed)
    out = []
    for it in range(n):
        nodes = rng.choice([1, 1, 1, 2])
        gpus = rng.randint(2, 8 if nodes == 1 else 4)
        nics = rng.randint(1, gpus) if nodes > 1 else 0
        fabric = rng.choice(["alltoall", "nvswitch"])
        ranks = nodes * gpus
        nv = rng.choice([120.0, 900.0])
        wl = rng.randint(0, 4)
        if wl == 0:
            w = {"kind": "skewed", "size": rng.randint(1, 300) * MiB, "ratio": rng.randint(0, 10) / 10,
                 "hot": rng.randrange(ranks)}
        elif wl == 1:
            w = {"kind": "irregular", "size": rng.randint(1, 1024) * MiB + rng.randint(0, 4095),
                 "sparsity": rng.randint(2, 10) / 10, "seed": it}
        elif wl == 2:
            w = {"kind": "stencil", "size": rng.randint(1, 128) * MiB}
        elif wl == 3:
            s = rng.randrange(ranks)
            d = (s + 1 + rng.randrange(ranks - 1)) % ranks
            w = {"kind": "p2p", "src": s, "dst": d, "size": rng.randint(1, 1024) * MiB + rng.randint(0, 7)}
        else:
            k = rng.randint(1, max(1, ranks // 2))
            w = {"kind": "aggregator", "dsts": rng.sample(range(ranks), k),
                 "size": rng.randint(1, 256) * MiB}
        planner = {"epsilon": rng.randint(1, 8) * MiB, "lambda": rng.randint(3, 10) / 10}
        if rng.random() < 0.2:
            planner["unpenalized"] = True
        if rng.random() < 0.1:
            planner["max_pair_visits"] = rng.randint(1, 20)
        out.append((f"fuzz{it}", {"ranks": ranks, "ranks_per_node": gpus,
                                  "topology": topo(gpus, fabric, nodes, nics, nv),
                                  "workload": w, "planner": planner}))
    return out


def transfer_requests():
    out = []
    rng = random.Random(7007)
    for it in range(40):
        hops = rng.randint(1, 4)
        chain = [[rng.uniform(20e9, 900e9), rng.uniform(0, 2e-6)] for _ in range(hops)]
        chunk = 64 * KiB * rng.randint(4, 8)
        slots = rng.randint(2, 20)
        out.append((f"tr{it}", {"chain": chain, "bytes": float(chunk * rng.randint(1, 60) + rng.randint(0, 999)),
                                "pipeline": {"pipe_chunk": chunk, "p2p_buffer": chunk * slots,
                                             "hop_latency": 0.0}}))
    return out


def main():
    configs = []
    for name, req in config_requests():
        r = dict(req, op="simulate")
        resp = ref.call(r)
        configs.append({"name": name, "request": req, "response": resp})
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(configs, f, separators=(",", ":"))

    fuzz = []
    for name, req in fuzz_requests(300, 2604):
        resp = ref.call(dict(req, op="plan"))
        fuzz.append({"name": name, "request": req, "response": resp})
    with open(os.path.join(HERE, "fuzz_plans.json"), "w") as f:
        json.dump(fuzz, f, separators=(",", ":"))

    trs = []
    for name, req in transfer_requests():
        resp = ref.call(dict(req, op="transfer"))
        trs.append({"name": name, "request": req,
                    "response": {"completion": resp["completion"],
                                 "start": resp["start"], "tx_done": resp["tx_done"]}})
    with open(os.path.join(HERE, "transfers.json"), "w") as f:
        json.dump(trs, f, separators=(",", ":"))

    topos = []
    for t in (topo(8, "nvswitch"), topo(4, "alltoall"), topo(4, "alltoall", 2, 2, 120.0),
              topo(2, "nvswitch", 2, 1, 120.0)):
        topos.append({"topology": t, "response": ref.call({"op": "topology", "topology": t})})
    with open(os.path.join(HERE, "topologies.json"), "w") as f:
        json.dump(topos, f, separators=(",", ":"))
    print("configs", len(configs), "fuzz", len(fuzz), "transfers", len(trs))


if __name__ == "__main__":
    main()
