"""Replay helpers: turn a golden request (tests/golden/*.json) into inputs for
the Python oracle and for the product's C ABI."""
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def matrix_for(mod, req):
    """Generate the request's demand matrix with module `mod` (oracle or product)."""
    w, R = req["workload"], req["ranks"]
    k = w["kind"]
    if k == "p2p":
        return mod.gen_p2p(R, w.get("src", 0), w.get("dst", 1), w["size"])
    if k == "skewed":
        return mod.gen_skewed_a2av(R, w["size"], w["ratio"], w.get("hot", 0))
    if k == "irregular":
        return mod.gen_irregular(R, w["size"], w["sparsity"], w["seed"])
    if k == "stencil":
        return mod.gen_stencil_1d(R, w["size"])
    if k == "aggregator":
        return mod.gen_aggregator(R, w["dsts"], w["size"])
    raise ValueError(k)


def topology_for(mod, req):
    t = req["topology"]
    return mod.build_canonical(t["nodes"], t["gpus"], t["nics"], mod.gbps(t["nvlink_gbps"]),
                               mod.gbps(t["rail_gbps"]), t["fabric"])


def config_for(mod, req):
    p = req.get("planner", {})
    cfg = mod.PlannerConfig()
    if "lambda" in p:
        cfg.lam = p["lambda"]
    if "epsilon" in p:
        cfg.epsilon = p["epsilon"]
    if p.get("unpenalized"):
        cfg.cost = mod.CostModel.unpenalized()
    if "max_pair_visits" in p:
        cfg.max_pair_visits = p["max_pair_visits"]
    return cfg


def rpn(req):
    return req.get("ranks_per_node", req["topology"]["gpus"])


def ref_flows(resp):
    """[(candidate, bytes), ...] per pair, from a reference plan response."""
    out = []
    for pp, cands in zip(resp["plan"]["pairs"], resp["flow_candidates"]):
        out.append([(c, f["bytes"]) for c, f in zip(cands, pp["flows"])])
    return out


def ref_stats(resp):
    st = dict(resp["plan"]["stats"])
    st.pop("wall_seconds", None)
    return st
