"""Planner quality against the exhaustive optimum (SURVEY.md sec. 8(f) row 4:
solve_exact as the quality referee for planner changes).

Restates the reference's acceptance criterion 1 (proj/tests/acceptance.cpp:58-117)
for the PRODUCT planner.  On instances small enough to solve exactly (the
reference's solve_exact through oracle/_ref, proj/src/oracle.cpp:67-91), the
unpenalized plan stays within 1.25x of the optimum and never loses to the
direct baseline.  Instances have the reference's shape -- a mesh of 2-4 GPUs,
or 2 nodes x 2 GPUs x 2 rails; 1-3 demands of 1-8 chunks of 4 MiB -- drawn with
Python's random (seed 1001), not libstdc++'s distributions.
"""
import random

import pytest

from oracle import ref
from paper_2604_00317_b200 import planner as P

MiB = 1 << 20
EPS = 4 * MiB
GAP_CAP = 1.25

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref (the compiled reference) is not built")


def _instances(n, seed=1001):
    rng = random.Random(seed)
    for _ in range(n):
        if rng.randint(0, 1):
            nodes, g, nics = 2, 2, 2
        else:
            nodes, g, nics = 1, rng.randint(2, 4), 0
        ranks = nodes * g
        nd = min(rng.randint(1, 3), ranks * (ranks - 1))
        m = [0] * (ranks * ranks)
        used = set()
        while len(used) < nd:
            s, d = rng.randrange(ranks), rng.randrange(ranks)
            if s == d or (s, d) in used:
                continue
            used.add((s, d))
            m[s * ranks + d] = rng.randint(1, 8) * EPS
        yield nodes, g, nics, ranks, m


def test_planner_within_gap_of_exact_optimum_and_never_worse_than_direct():
    worst = 1.0
    for nodes, g, nics, ranks, m in _instances(300):
        topo = P.build_canonical(nodes, g, nics, 120e9, 50e9, P.ALLTOALL)
        cfg = P.PlannerConfig(cost=P.CostModel.unpenalized())
        got = P.max_normalized_load(P.plan(topo, ranks, g, m, cfg))
        base = P.max_normalized_load(P.plan_direct_baseline(topo, ranks, g, m))
        z = ref.call({"op": "exact", "ranks": ranks, "ranks_per_node": g, "epsilon": EPS,
                      "topology": {"nodes": nodes, "gpus": g, "nics": nics, "fabric": "alltoall",
                                   "nvlink_gbps": 120.0, "rail_gbps": 50.0},
                      "workload": {"kind": "matrix", "bytes": m}})["z_star"]
        gap = got / z
        worst = max(worst, gap)
        assert gap <= GAP_CAP + 1e-9, (nodes, g, m, got, z)
        assert got <= base * (1 + 1e-12), (nodes, g, m, got, base)
    assert worst >= 1.0 - 1e-12  # the exact optimum is a lower bound
