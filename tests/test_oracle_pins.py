"""Pin the oracle (oracle/nimble_oracle.py) before trusting it.

1. The reference's own known-answer tests for this path (proj/tests/*.cpp),
   restated against the oracle.
2. Every golden fixture dumped from the compiled reference (tests/golden/).
3. When the compiled reference is present (build container), fresh random
   instances compared live against oracle/_ref.
"""
import math
import os
import random

import pytest

from oracle import nimble_oracle as O
from tests import _cases

MiB, KiB = O.MiB, O.KiB


# ---- 1. reference known-answer tests -------------------------------------

def test_units():  # proj/include/nimble/units.hpp:7-12
    assert (O.KiB, O.MiB, O.GiB) == (1024, 1 << 20, 1 << 30)
    assert O.gbps(120) == 120e9


def test_skew_goldens():  # proj/tests/test_workloads.cpp:19-43
    d = O.gen_skewed_a2av(4, 12, 0.5, 3)
    for s in range(3):
        assert d[s * 4 + 3] == 6 and sum(d[s * 4:(s + 1) * 4]) == 12
    assert d[0 * 4 + 1] == 3 and d[0 * 4 + 2] == 3
    assert d[3 * 4 + 0] == d[3 * 4 + 1] == d[3 * 4 + 2] == 4
    e = O.gen_skewed_a2av(4, 10, 0.5, 0)
    assert (e[1 * 4 + 0], e[1 * 4 + 2], e[1 * 4 + 3]) == (5, 2, 3)
    with pytest.raises(ValueError):
        O.gen_skewed_a2av(4, 12, 1.5, 0)
    with pytest.raises(ValueError):
        O.gen_skewed_a2av(4, 12, 0.5, 4)


def test_per_sender_hot():  # test_workloads.cpp:45-52
    d = O.gen_skewed_a2av(4, 12, 1.0, 1, 0, True)
    assert d[0 * 4 + 1] == d[1 * 4 + 2] == d[2 * 4 + 3] == d[3 * 4 + 0] == 12


def test_irregular_seed42_frozen():  # test_workloads.cpp:81-100
    d = O.gen_irregular(4, 1000000, 0.5, 42)
    assert sum(d) == 1000000
    assert d[1 * 4 + 0] == 159477 and d[1 * 4 + 3] == 148322 and d[2 * 4 + 1] == 192356
    assert d[2 * 4 + 3] == 220084 and d[3 * 4 + 0] == 175289 and d[3 * 4 + 1] == 104472
    assert d[1] + d[2] + d[3] == 0
    assert O.gen_irregular(4, 1000000, 0.5, 42) == d
    assert O.gen_irregular(4, 1000000, 0.5, 43) != d


def test_stencil_and_aggregator():  # test_workloads.cpp:54-79
    d = O.gen_stencil_1d(4, 7)
    assert d[0 * 4 + 1] == d[1 * 4 + 0] == d[1 * 4 + 2] == d[2 * 4 + 3] == d[3 * 4 + 2] == 7
    assert d[0 * 4 + 3] == d[3 * 4 + 0] == 0 and sum(d) == 42
    a = O.gen_aggregator(5, [1, 3], 10)
    for s in (0, 2, 4):
        assert a[s * 5 + 1] == a[s * 5 + 3] == 5
    assert O.gen_aggregator(4, [1, 1], 10)[0 * 4 + 1] == 10


def test_candidates_mesh_and_nvswitch():  # test_planner.cpp:33-58
    t = O.build_canonical(1, 4, 0, O.gbps(120), O.gbps(50), O.ALLTOALL)
    c = O.enumerate_paths(t, 4, 4, 0, 1)
    assert [x.cls for x in c] == [O.DIRECT, O.TWO_HOP, O.TWO_HOP]
    assert c[0].edges == [t.nvlink_id(0, 0, 1)]
    assert c[1].via == 2 and c[1].edges == [t.nvlink_id(0, 0, 2), t.nvlink_id(0, 2, 1)]
    assert c[2].via == 3
    s = O.build_canonical(1, 8, 0, O.gbps(120), O.gbps(50), O.NVSWITCH)
    c = O.enumerate_paths(s, 8, 8, 2, 6)
    assert len(c) == 1 and c[0].edges == [s.port_up_id(0, 2), s.port_down_id(0, 6)]


def test_rails_destination_matched():  # test_planner.cpp:60-78
    t = O.build_canonical(2, 4, 2, O.gbps(120), O.gbps(50), O.ALLTOALL)
    c = O.enumerate_paths(t, 8, 4, 0, 5)
    assert len(c) == 2 and c[0].rail == 1 and c[0].pair_direct and c[0].hops == 1
    assert c[0].edges == [t.nvlink_id(0, 0, 1), t.attach_up_id(0, 1), t.rail_id(0, 1, 1), t.attach_down_id(1, 1)]
    assert c[1].rail == 0 and c[1].hops == 2


def test_hop_penalty():  # test_planner.cpp:80-94
    cost = O.CostModel()
    via = O.Candidate(O.TWO_HOP, hops=2)
    assert math.isinf(cost.hop_penalty(via, MiB)) and math.isinf(cost.hop_penalty(via, 512 * KiB))
    assert cost.hop_penalty(via, 32 * MiB) == pytest.approx(0.125)
    assert cost.hop_penalty(via, 64 * MiB) == 0.0 and cost.hop_penalty(via, 256 * MiB) == 0.0
    assert cost.hop_penalty(O.Candidate(O.DIRECT), KiB) == 0.0
    assert O.CostModel.unpenalized().hop_penalty(via, KiB) == 0.0


def test_golden_split_88_84_84():  # test_planner.cpp:96-111
    t = O.build_canonical(1, 4, 0, O.gbps(120), O.gbps(50), O.ALLTOALL)
    p = O.plan(t, 4, 4, O.gen_p2p(4, 0, 1, 256 * MiB))
    assert [b for _, b in p.pairs[0].flows] == [88.0 * MiB, 84.0 * MiB, 84.0 * MiB]
    assert p.pairs[0].flows[0][0] == 0
    assert p.stats["pair_visits"] == 7 and p.stats["placements"] == 64
    assert O.max_normalized_load(t, p) == 88.0 * MiB / O.gbps(120)


def test_small_messages_direct():  # test_planner.cpp:113-122
    t = O.build_canonical(1, 4, 0, O.gbps(120), O.gbps(50), O.ALLTOALL)
    for size in (64 * KiB, 512 * KiB, MiB):
        p = O.plan(t, 4, 4, O.gen_p2p(4, 0, 1, size))
        assert p.pairs[0].flows == [(0, float(size))]


def test_refinement_never_loses():  # test_planner.cpp:141-158
    t = O.build_canonical(2, 2, 2, O.gbps(120), O.gbps(50), O.ALLTOALL)
    m = [0] * 16
    m[2 * 4 + 3] = 28 * MiB
    m[1 * 4 + 3] = 8 * MiB
    cfg = O.PlannerConfig(cost=O.CostModel.unpenalized())
    p = O.plan(t, 4, 2, m, cfg)
    base = O.plan_direct_baseline(t, 4, 2, m)
    assert O.max_normalized_load(t, p) == pytest.approx(28.0 * MiB / O.gbps(120), rel=1e-12)
    assert O.max_normalized_load(t, p) <= O.max_normalized_load(t, base)


def test_visit_budget_fallback():  # test_planner.cpp:160-169
    t = O.build_canonical(1, 4, 0, O.gbps(120), O.gbps(50), O.ALLTOALL)
    p = O.plan(t, 4, 4, O.gen_skewed_a2av(4, 64 * MiB, 0.5, 0), O.PlannerConfig(max_pair_visits=3))
    assert p.stats["fallback_pairs"] > 0
    for pp in p.pairs:
        assert sum(b for _, b in pp.flows) == pp.demand


def test_config_validation():  # test_planner.cpp:193-205
    t = O.build_canonical(1, 4, 0, O.gbps(120), O.gbps(50), O.ALLTOALL)
    m = O.gen_p2p(4, 0, 1, MiB)
    for bad in (O.PlannerConfig(lam=0.0), O.PlannerConfig(lam=1.5), O.PlannerConfig(epsilon=0)):
        with pytest.raises(ValueError):
            O.plan(t, 4, 4, m, bad)


def test_pipeline_recurrence():  # proj/tests/test_pipeline.cpp:27-89
    tau = 512.0 * KiB / 1e9
    c, *_ = O.simulate_transfer([(1e9, 2e-6), (1e9, 2e-6)], 4 * MiB)
    assert c == pytest.approx(9 * tau + 4e-6, rel=1e-14)
    c, start, txd, _ = O.simulate_transfer([(4e9, 0.0), (1e9, 0.0)], 8 * MiB, p2p_buffer=MiB)
    S = O.slots(MiB)
    assert S == 2 and len(start[0]) == 16
    for k in range(S, 16):
        assert start[0][k] >= txd[1][k - S]
    assert c == pytest.approx(8 * MiB / 1e9 + 512.0 * KiB / 4e9)
    assert O.chunk_sizes(512 * KiB + 100, 512 * KiB) == [512 * KiB, 100]


def test_port_bound_c3():  # c3 r=0.7 bound 1.4615 ms
    m = O.gen_skewed_a2av(8, 256 * MiB, 0.7, 0)
    assert O.port_bound_seconds(m, 8, 900e9) == pytest.approx(1.4615e-3, rel=1e-4)
    t = O.build_canonical(1, 8, 0, 900e9, 0, O.NVSWITCH)
    assert O.max_normalized_load(t, O.plan_direct_baseline(t, 8, 8, m)) == O.port_bound_seconds(m, 8, 900e9)


# ---- 2. golden fixtures from the compiled reference -----------------------

@pytest.mark.parametrize("fixture", ["configs.json", "fuzz_plans.json"])
def test_oracle_matches_reference_fixtures(fixture):
    for case in _cases.load(fixture):
        req, resp = case["request"], case["response"]
        t = _cases.topology_for(O, req)
        m = _cases.matrix_for(O, req)
        assert m == resp["matrix"], case["name"]
        p = O.plan(t, req["ranks"], _cases.rpn(req), m, _cases.config_for(O, req))
        assert [pp.flows for pp in p.pairs] == [[(c, b) for c, b in f] for f in _cases.ref_flows(resp)], case["name"]
        assert O.plan_link_loads(t, p) == resp["loads"], case["name"]
        assert p.stats == _cases.ref_stats(resp), case["name"]


def test_oracle_matches_reference_transfers():
    for case in _cases.load("transfers.json"):
        req, resp = case["request"], case["response"]
        pl = req["pipeline"]
        c, start, txd, _ = O.simulate_transfer([tuple(h) for h in req["chain"]], int(req["bytes"]),
                                               pipe_chunk=pl["pipe_chunk"], p2p_buffer=pl["p2p_buffer"])
        assert c == resp["completion"], case["name"]
        assert start == resp["start"] and txd == resp["tx_done"], case["name"]


def test_oracle_topology_ids_match_reference():
    for case in _cases.load("topologies.json"):
        t = case["topology"]
        topo = O.build_canonical(t["nodes"], t["gpus"], t["nics"], O.gbps(t["nvlink_gbps"]),
                                 O.gbps(t["rail_gbps"]), t["fabric"])
        assert topo.capacity == [l["capacity"] for l in case["response"]["links"]]


# ---- 3. live against the compiled reference (build container only) --------

def _ref_available():
    from oracle import ref
    return ref.available()


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built (reference absent)")
def test_oracle_matches_live_reference_random():
    from oracle import ref
    rng = random.Random(99)
    for it in range(60):
        gpus = rng.randint(2, 8)
        fabric = rng.choice([O.ALLTOALL, O.NVSWITCH])
        req = {"ranks": gpus, "topology": {"nodes": 1, "gpus": gpus, "nics": 0, "fabric": fabric,
                                           "nvlink_gbps": 900.0, "rail_gbps": 50.0},
               "workload": {"kind": "skewed", "size": rng.randint(1, 400) * MiB + rng.randint(0, 99),
                            "ratio": rng.random(), "hot": rng.randrange(gpus)},
               "planner": {"epsilon": rng.randint(1, 8) * MiB, "lambda": rng.randint(2, 10) / 10}}
        resp = ref.call(dict(req, op="plan"))
        t = _cases.topology_for(O, req)
        m = _cases.matrix_for(O, req)
        assert m == resp["matrix"]
        p = O.plan(t, gpus, gpus, m, _cases.config_for(O, req))
        assert [pp.flows for pp in p.pairs] == [[(c, b) for c, b in f] for f in _cases.ref_flows(resp)]
        assert O.plan_link_loads(t, p) == resp["loads"]
