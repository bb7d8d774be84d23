"""Parity of the product's planning path (C ABI, host C++) with the reference.

Bit-exact chunk-to-path assignments and stats, link loads exact (the bar is
1e-6 relative; they are integers, so exact), for:
  - every golden fixture dumped from the compiled reference (BASELINE configs
    c1..c5 on both fabric models, and a 300-instance fuzz corpus);
  - fresh random instances against the Python oracle;
  - the reference's own unit-test vectors, re-run through the product API.
"""
import json
import math
import random

import pytest

from oracle import nimble_oracle as O
from paper_2604_00317_b200 import planner as P
from paper_2604_00317_b200._lib import NimbleError
from tests import _cases

MiB, KiB = P.MiB, P.KiB


def _product_plan(req):
    t = _cases.topology_for(P, req)
    m = _cases.matrix_for(P, req)
    return t, m, P.plan(t, req["ranks"], _cases.rpn(req), m, _cases.config_for(P, req))


@pytest.mark.parametrize("fixture", ["configs.json", "fuzz_plans.json"])
def test_product_matches_reference_fixtures(lib, fixture):
    for case in _cases.load(fixture):
        req, resp = case["request"], case["response"]
        t, m, p = _product_plan(req)
        assert m == resp["matrix"], case["name"]
        assert [pp.flows for pp in p.pairs] == [[(c, b) for c, b in f] for f in _cases.ref_flows(resp)], case["name"]
        loads = p.link_loads
        for a, b in zip(loads, resp["loads"]):
            assert a == b or abs(a - b) <= 1e-6 * abs(b), case["name"]
        assert p.max_normalized_load == resp["max_norm_load"], case["name"]
        assert {k: v for k, v in p.stats.items() if k != "wall_seconds"} == _cases.ref_stats(resp), case["name"]
        # plan_to_json fields (planner.cpp:466-492)
        j = json.loads(p.json)
        want = resp["plan"]
        assert j["epsilon"] == want["epsilon"]
        assert [[(f["class"], f["via"], f["rail"], f["bytes"]) for f in pp["flows"]] for pp in j["pairs"]] == \
               [[(f["class"], f["via"], f["rail"], f["bytes"]) for f in pp["flows"]] for pp in want["pairs"]]
        assert [(pp["src"], pp["dst"], pp["demand"]) for pp in j["pairs"]] == \
               [(pp["src"], pp["dst"], pp["demand"]) for pp in want["pairs"]]


def test_product_direct_baseline_matches_reference(lib):
    for case in _cases.load("configs.json"):
        req, resp = case["request"], case["response"]
        t = _cases.topology_for(P, req)
        m = _cases.matrix_for(P, req)
        b = P.plan_direct_baseline(t, req["ranks"], _cases.rpn(req), m)
        assert b.max_normalized_load == resp["direct_max_norm_load"], case["name"]


def test_product_matches_oracle_random(lib):
    rng = random.Random(4242)
    for it in range(120):
        gpus = rng.randint(2, 8)
        fabric = rng.choice([P.ALLTOALL, P.NVSWITCH])
        R = rng.randint(2, gpus)
        kind = rng.choice(["skewed", "irregular", "p2p", "stencil"])
        w = {"kind": kind, "size": rng.randint(1, 512) * MiB + rng.randint(0, 4095)}
        if kind == "skewed":
            w.update(ratio=rng.random(), hot=rng.randrange(R))
        elif kind == "irregular":
            w.update(sparsity=rng.randint(1, 10) / 10, seed=it)
        elif kind == "p2p":
            w.update(src=0, dst=R - 1)
        req = {"ranks": R, "ranks_per_node": gpus,
               "topology": {"nodes": 1, "gpus": gpus, "nics": 0, "fabric": fabric,
                            "nvlink_gbps": rng.choice([120.0, 900.0]), "rail_gbps": 50.0},
               "workload": w, "planner": {"epsilon": rng.randint(1, 8) * MiB, "lambda": rng.randint(1, 10) / 10}}
        to = _cases.topology_for(O, req)
        mo = _cases.matrix_for(O, req)
        po = O.plan(to, R, gpus, mo, _cases.config_for(O, req))
        t, m, p = _product_plan(req)
        assert m == mo
        assert [pp.flows for pp in p.pairs] == [pp.flows for pp in po.pairs], req
        assert p.link_loads == O.plan_link_loads(to, po)
        assert {k: v for k, v in p.stats.items() if k != "wall_seconds"} == po.stats


# ---- the reference's unit tests, through the product API -----------------

def test_mesh_candidates(lib):  # test_planner.cpp:33-49
    t = P.build_canonical(1, 4, 0, P.gbps(120), P.gbps(50), P.ALLTOALL)
    c = P.enumerate_paths(t, 4, 4, 0, 1)
    assert [x.cls for x in c] == ["direct", "intra_two_hop", "intra_two_hop"]
    assert c[0].edges == [t.nvlink_id(0, 0, 1)] and c[0].hops == 1
    assert c[1].via == 2 and c[1].hops == 2 and c[1].edges == [t.nvlink_id(0, 0, 2), t.nvlink_id(0, 2, 1)]
    assert c[2].via == 3
    with pytest.raises(NimbleError):
        P.enumerate_paths(t, 4, 4, 1, 1)
    with pytest.raises(NimbleError):
        P.enumerate_paths(t, 4, 4, 0, 7)


def test_nvswitch_has_no_detours(lib):  # test_planner.cpp:51-58
    t = P.build_canonical(1, 8, 0, P.gbps(120), P.gbps(50), P.NVSWITCH)
    c = P.enumerate_paths(t, 8, 8, 2, 6)
    assert len(c) == 1 and c[0].cls == "direct"
    assert c[0].edges == [t.port_up_id(0, 2), t.port_down_id(0, 6)]


def test_rails_destination_matched(lib):  # test_planner.cpp:60-78
    t = P.build_canonical(2, 4, 2, P.gbps(120), P.gbps(50), P.ALLTOALL)
    c = P.enumerate_paths(t, 8, 4, 0, 5)
    assert len(c) == 2 and c[0].cls == "inter_rail" and c[0].rail == 1 and c[0].hops == 1
    assert c[0].edges == [t.nvlink_id(0, 0, 1), t.attach_up_id(0, 1), t.rail_id(0, 1, 1), t.attach_down_id(1, 1)]
    assert c[1].rail == 0 and c[1].hops == 2
    assert c[1].edges == [t.attach_up_id(0, 0), t.rail_id(0, 1, 0), t.attach_down_id(1, 0), t.nvlink_id(1, 0, 1)]
    with pytest.raises(NimbleError):
        P.enumerate_paths(P.build_canonical(2, 2, 0, P.gbps(100), P.gbps(50), P.ALLTOALL), 4, 2, 0, 2)


def test_golden_split(lib):  # test_planner.cpp:96-111
    t = P.build_canonical(1, 4, 0, P.gbps(120), P.gbps(50), P.ALLTOALL)
    p = P.plan(t, 4, 4, P.gen_p2p(4, 0, 1, 256 * MiB))
    assert p.pairs[0].flows == [(0, 88.0 * MiB), (1, 84.0 * MiB), (2, 84.0 * MiB)]
    assert p.stats["pair_visits"] == 7 and p.stats["placements"] == 64
    assert p.max_normalized_load == 88.0 * MiB / P.gbps(120)


def test_small_messages_direct(lib):  # test_planner.cpp:113-122
    t = P.build_canonical(1, 4, 0, P.gbps(120), P.gbps(50), P.ALLTOALL)
    for size in (64 * KiB, 512 * KiB, MiB):
        assert P.plan(t, 4, 4, P.gen_p2p(4, 0, 1, size)).pairs[0].flows == [(0, float(size))]


def test_deterministic(lib):  # test_planner.cpp:124-139
    t = P.build_canonical(2, 4, 4, P.gbps(120), P.gbps(50), P.ALLTOALL)
    m = P.gen_skewed_a2av(8, 128 * MiB, 0.7, 0)
    a, b = P.plan(t, 8, 4, m), P.plan(t, 8, 4, m)
    assert [pp.flows for pp in a.pairs] == [pp.flows for pp in b.pairs]


def test_refinement_never_loses(lib):  # test_planner.cpp:141-158
    t = P.build_canonical(2, 2, 2, P.gbps(120), P.gbps(50), P.ALLTOALL)
    m = [0] * 16
    m[2 * 4 + 3] = 28 * MiB
    m[1 * 4 + 3] = 8 * MiB
    p = P.plan(t, 4, 2, m, P.PlannerConfig(cost=P.CostModel.unpenalized()))
    base = P.plan_direct_baseline(t, 4, 2, m)
    assert p.max_normalized_load == pytest.approx(28.0 * MiB / P.gbps(120), rel=1e-12)
    assert p.max_normalized_load <= base.max_normalized_load


def test_visit_budget_fallback(lib):  # test_planner.cpp:160-169
    t = P.build_canonical(1, 4, 0, P.gbps(120), P.gbps(50), P.ALLTOALL)
    p = P.plan(t, 4, 4, P.gen_skewed_a2av(4, 64 * MiB, 0.5, 0), P.PlannerConfig(max_pair_visits=3))
    assert p.stats["fallback_pairs"] > 0
    for pp in p.pairs:
        assert sum(b for _, b in pp.flows) == pp.demand


def test_config_validation(lib):  # test_planner.cpp:193-205
    t = P.build_canonical(1, 4, 0, P.gbps(120), P.gbps(50), P.ALLTOALL)
    m = P.gen_p2p(4, 0, 1, MiB)
    for bad in (P.PlannerConfig(lam=0.0), P.PlannerConfig(lam=1.5), P.PlannerConfig(epsilon=0)):
        with pytest.raises(NimbleError) as e:
            P.plan(t, 4, 4, m, bad)
        assert e.value.code == 4  # nimbleInvalidArgument


def test_workload_errors(lib):  # test_workloads.cpp:10-43,121-131
    with pytest.raises(NimbleError):
        P.gen_p2p(4, 1, 1, MiB)
    with pytest.raises(NimbleError):
        P.gen_p2p(4, 0, 4, MiB)
    with pytest.raises(NimbleError):
        P.gen_skewed_a2av(4, 12, 1.5, 0)
    with pytest.raises(NimbleError):
        P.gen_skewed_a2av(4, 12, 0.5, 4)
    with pytest.raises(NimbleError):
        P.gen_aggregator(4, [], 10)
    with pytest.raises(NimbleError):
        P.gen_irregular(4, 10, 0.0, 1)
    t = P.build_canonical(1, 2, 0, P.gbps(100), P.gbps(50), P.ALLTOALL)
    with pytest.raises(NimbleError):  # nonzero diagonal
        P.plan(t, 2, 2, [5, 1, 2, 0])


def test_irregular_seed42(lib):  # test_workloads.cpp:81-100
    d = P.gen_irregular(4, 1000000, 0.5, 42)
    assert sum(d) == 1000000 and d[4] == 159477 and d[7] == 148322 and d[9] == 192356
    assert d[11] == 220084 and d[12] == 175289 and d[13] == 104472


def test_payload_matrix_roundtrip(lib):  # test_workloads.cpp:102-110
    d = P.gen_irregular(6, 12345678, 0.4, 7)
    back, R = P.read_payload_matrix(P.write_payload_matrix(d, 6))
    assert R == 6 and back == d
    for bad in ("1 2\n3 4 5\n", "0 1\nx 0\n", "1 1\n1 0\n"):
        with pytest.raises(NimbleError):
            P.read_payload_matrix(bad)


def test_topology_inventory_and_files(lib):  # test_topology.cpp:10-105
    t = P.build_canonical(2, 4, 4, P.gbps(120), P.gbps(50), P.ALLTOALL)
    assert t.link_count() == 24 + 16 + 8
    s = P.build_canonical(1, 8, 0, P.gbps(120), P.gbps(50), P.NVSWITCH)
    assert s.link_count() == 16 and s.link(s.port_up_id(0, 3))["name"] == "n0.g3->n0.sw"
    pair = P.build_canonical(2, 2, 2, P.gbps(120), P.gbps(50), P.ALLTOALL)
    text = pair.save()
    assert P.load_topology(text).save() == text
    one = P.build_canonical(1, 2, 0, P.gbps(100), P.gbps(50), P.ALLTOALL)
    one.set_capacity(0, P.gbps(75))
    back = P.load_topology(one.save())
    assert back.capacities == [P.gbps(75), P.gbps(100)]
    with pytest.raises(NimbleError):
        P.load_topology("nodes 1\n")
    with pytest.raises(NimbleError):
        P.load_topology(pair.save() + "link n0.nic0 n1.nic1 10\n")
    for args in ((0, 4, 0, 1e9, 1e9), (2, 2, 3, 1e9, 1e9), (1, 2, 0, 0.0, 1e9), (2, 4, 4, 1e11, 0.0)):
        with pytest.raises(NimbleError):
            P.build_canonical(*args, P.ALLTOALL)


def test_topology_ids_match_reference(lib):
    for case in _cases.load("topologies.json"):
        t = case["topology"]
        topo = P.build_canonical(t["nodes"], t["gpus"], t["nics"], P.gbps(t["nvlink_gbps"]),
                                 P.gbps(t["rail_gbps"]), t["fabric"])
        want = case["response"]["links"]
        assert [topo.link(i)["name"] for i in range(topo.link_count())] == [l["name"] for l in want]
        assert topo.save() == case["response"]["text"]


def test_port_bound_is_direct_max_load(lib):
    for r in (0.0, 0.3, 0.7, 0.9):
        m = P.gen_skewed_a2av(8, 256 * MiB, r, 0)
        t = P.build_canonical(1, 8, 0, 900e9, 0, P.NVSWITCH)
        assert P.plan_direct_baseline(t, 8, 8, m).max_normalized_load == P.port_bound_seconds(m, 8, 900e9)
    assert P.port_bound_seconds(P.gen_skewed_a2av(8, 256 * MiB, 0.7, 0), 8) == pytest.approx(1.4615e-3, rel=1e-4)
    assert not math.isnan(P.port_bound_seconds([0, 0, 0, 0], 2))


def test_plan_json_round_trip(lib):  # test_planner.cpp:171-191
    t = P.build_canonical(2, 4, 4, P.gbps(120), P.gbps(50), P.ALLTOALL)
    m = P.gen_irregular(8, 512 * MiB, 0.5, 3)
    p = P.plan(t, 8, 4, m)
    back = P.plan_from_json(t, 8, 4, p.json)
    assert [pp.flows for pp in back.pairs] == [pp.flows for pp in p.pairs]
    assert back.stats["placements"] == p.stats["placements"]
    assert back.link_loads == p.link_loads
    doc = P.plan_to_json(p)
    doc["pairs"][0]["flows"][0]["bytes"] = 1.0  # break conservation
    with pytest.raises(NimbleError):
        P.plan_from_json(t, 8, 4, doc)


def test_plan_from_reference_json(lib):
    """The reference's own plan.json documents (dumped by oracle/_ref) load into
    the product with identical flows and loads."""
    for case in _cases.load("configs.json"):
        req, resp = case["request"], case["response"]
        t = _cases.topology_for(P, req)
        back = P.plan_from_json(t, req["ranks"], _cases.rpn(req), resp["plan"])
        assert [pp.flows for pp in back.pairs] == [[(c, b) for c, b in f] for f in _cases.ref_flows(resp)]
        assert back.link_loads == resp["loads"]


def test_nvswitch_mcf_plan_equals_direct_plan_flows(lib):
    """The communicator plans nvswitch exchanges with the direct plan (comm.cpp
    plan_for): with one candidate per pair the MCF sweep has no choice, so its
    flows must equal the direct plan's on any matrix."""
    import random
    rng = random.Random(5)
    for R in (2, 3, 4, 8):
        topo = P.build_canonical(1, R, 0, 900e9, 0, P.NVSWITCH)
        for _ in range(100):
            m = [0 if i // R == i % R else rng.choice([0, rng.randint(1, 1 << 30), rng.randint(1, 1 << 20)])
                 for i in range(R * R)]
            a = P.plan(topo, R, R, m)
            b = P.plan_direct_baseline(topo, R, R, m)
            assert [(p.src, p.dst, p.flows) for p in a.pairs] == [(p.src, p.dst, p.flows) for p in b.pairs]
