"""Planner latency: the product's plan() vs the reference's (Table II protocol,
5 warm-up + median of 100 calls, tools/nimble.cpp:385-403), single host core.
Writes profiles/r01_planner_latency.md.  Needs oracle/_ref (build container)."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20
CASES = [
    ("c3 nvswitch8 r=0.7", 8, "nvswitch", lambda: P.gen_skewed_a2av(8, 256 * MiB, 0.7, 0)),
    ("c3 mesh8 r=0.7", 8, "alltoall", lambda: P.gen_skewed_a2av(8, 256 * MiB, 0.7, 0)),
    ("c4 nvswitch8 1 GiB", 8, "nvswitch", lambda: P.gen_irregular(8, 1 << 30, 0.5, 1)),
    ("c5 nvswitch8 uniform", 8, "nvswitch", lambda: P.gen_skewed_a2av(8, 256 * MiB, 1 / 7, 0)),
    ("c2 mesh4 p2p 1 GiB", 4, "alltoall", lambda: P.gen_p2p(4, 0, 1, 1 << 30)),
    ("stencil mesh8 64 MiB", 8, "alltoall", lambda: P.gen_stencil_1d(8, 64 * MiB)),
]


def main():
    rows = ["# Planner latency (round 1)", "",
            "- Protocol: `plan()` with 5 warm-up calls, then the median of 100 timed calls, on one host core.",
            "- Each side is repeated 5 times, interleaved, and the best median is kept (the host is shared).",
            "- Reference: its own `PlanStats.wall_seconds` (`planner.cpp:325,426`) through oracle/_ref.",
            "- Product: `nimblePlanCreate`, also timed by `PlanStats.wall_seconds`.",
            "- Both use the same matrix and produce the same (bit-exact) plan.", "",
            "| case | reference ms | product ms | speed-up |", "|---|---|---|---|"]
    for name, R, fab, gen in CASES:
        m = gen()
        req = {"ranks": R, "topology": {"nodes": 1, "gpus": R, "nics": 0, "fabric": fab, "nvlink_gbps": 900.0,
                                        "rail_gbps": 50.0}, "workload": {"kind": "matrix", "bytes": m}}
        topo = P.build_canonical(1, R, 0, 900e9, 0, fab)
        t_ref, t_prod = float("inf"), float("inf")
        for _ in range(5):  # interleaved repeats, best median of each: the host is shared and noisy
            t_ref = min(t_ref, ref.time_plan(req, 5, 100))
            for _ in range(5):
                P.plan(topo, R, R, m)
            t_prod = min(t_prod, statistics.median(P.plan(topo, R, R, m).stats["wall_seconds"] for _ in range(100)))
        rows.append(f"| {name} | {t_ref * 1e3:.4f} | {t_prod * 1e3:.4f} | {t_ref / t_prod:.2f}x |")
        print(rows[-1], flush=True)
    with open(os.path.join(ROOT, "profiles", "r01_planner_latency.md"), "w") as f:
        f.write("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
