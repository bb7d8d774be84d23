"""Host-side mirror of the reference's planning API, over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/nimble/{topology,workloads,planner}.hpp), so the
parity tests read like the reference's own tests.  Every function calls into
libnimble_b200.so; nothing is computed in Python.  Errors raise
`NimbleError` (a RuntimeError), where the reference throws
std::runtime_error / std::logic_error.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field

from . import _lib
from ._lib import c_double, c_int, c_size, c_u64, c_void_p

KiB = 1024
MiB = 1024 * KiB
GiB = 1024 * MiB

ALLTOALL, NVSWITCH = "alltoall", "nvswitch"
_FABRIC = {ALLTOALL: 0, NVSWITCH: 1}
ROUTE_NAMES = {0: "direct", 1: "intra_two_hop", 2: "inter_rail"}


def gbps(x: float) -> float:
    return x * 1e9


class Topology:
    """build_canonical() result (topology.hpp:41-70)."""

    def __init__(self, handle, nodes, gpus, nics, fabric):
        self._h = handle
        self.nodes, self.gpus_per_node, self.nics_per_node, self.fabric = nodes, gpus, nics, fabric

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib().nimbleTopologyDestroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def link_count(self) -> int:
        n = c_int()
        _lib.call("nimbleTopologyLinkCount", self._h, ctypes.byref(n))
        return n.value

    def link(self, i):
        kind, cap = c_int(), c_double()
        name = ctypes.create_string_buffer(64)
        _lib.call("nimbleTopologyLink", self._h, i, ctypes.byref(kind), ctypes.byref(cap), name, 64)
        return {"id": i, "kind": kind.value, "capacity": cap.value, "name": name.value.decode()}

    @property
    def capacities(self):
        return [self.link(i)["capacity"] for i in range(self.link_count())]

    def set_capacity(self, i, bytes_per_s):
        _lib.call("nimbleTopologySetCapacity", self._h, i, bytes_per_s)

    def _id(self, kind, node, a, b):
        out = c_int()
        _lib.call("nimbleTopologyLinkId", self._h, kind, node, a, b, ctypes.byref(out))
        return out.value

    def nvlink_id(self, node, a, b):
        return self._id(0, node, a, b)

    def port_up_id(self, node, g):
        return self._id(1, node, g, 0)

    def port_down_id(self, node, g):
        return self._id(1, node, g, 1)

    def attach_up_id(self, node, nic):
        return self._id(2, node, nic, 0)

    def attach_down_id(self, node, nic):
        return self._id(2, node, nic, 1)

    def rail_id(self, a, b, r):
        return self._id(3, a, b, r)

    def save(self) -> str:
        need = c_size()
        _lib.lib().nimbleTopologySave(self._h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        _lib.call("nimbleTopologySave", self._h, buf, need.value, ctypes.byref(need))
        return buf.value.decode()


def build_canonical(nodes, gpus_per_node, nics_per_node, nvlink_capacity, rail_capacity,
                    fabric=ALLTOALL) -> Topology:
    h = c_void_p()
    _lib.call("nimbleTopologyCreate", nodes, gpus_per_node, nics_per_node, float(nvlink_capacity),
              float(rail_capacity), _FABRIC[fabric], ctypes.byref(h))
    return Topology(h, nodes, gpus_per_node, nics_per_node, fabric)


def load_topology(text: str) -> Topology:
    h = c_void_p()
    _lib.call("nimbleTopologyLoad", text.encode(), ctypes.byref(h))
    t = Topology(h, 0, 0, 0, "")
    return t


# ------------------------------------------------------------------ workloads

def _matrix(ranks):
    return (c_u64 * (ranks * ranks))()


def gen_p2p(ranks, src, dst, size):
    m = _matrix(max(ranks, 1))
    _lib.call("nimbleGenP2P", ranks, src, dst, size, m)
    return list(m)


def gen_skewed_a2av(ranks, per_rank_bytes, ratio, hot_dst=0, seed=0, per_sender_hot=False):
    del seed  # stored only, never used by the generator (workloads.cpp:69)
    m = _matrix(max(ranks, 1))
    _lib.call("nimbleGenSkewed", ranks, per_rank_bytes, float(ratio), hot_dst, int(per_sender_hot), m)
    return list(m)


def gen_stencil_1d(ranks, halo_bytes):
    m = _matrix(max(ranks, 1))
    _lib.call("nimbleGenStencil1D", ranks, halo_bytes, m)
    return list(m)


def gen_aggregator(ranks, dsts, per_src_bytes):
    m = _matrix(max(ranks, 1))
    arr = (c_int * max(len(dsts), 1))(*dsts)
    _lib.call("nimbleGenAggregator", ranks, arr, len(dsts), per_src_bytes, m)
    return list(m)


def gen_irregular(ranks, total_bytes, sparsity, seed):
    m = _matrix(max(ranks, 1))
    _lib.call("nimbleGenIrregular", ranks, total_bytes, float(sparsity), seed, m)
    return list(m)


def write_payload_matrix(matrix, ranks) -> str:
    arr = _lib.u64_array(matrix)
    need = c_size()
    _lib.lib().nimbleMatrixToText(ranks, arr, None, 0, ctypes.byref(need))
    buf = ctypes.create_string_buffer(need.value)
    _lib.call("nimbleMatrixToText", ranks, arr, buf, need.value, ctypes.byref(need))
    return buf.value.decode()


def read_payload_matrix(text: str):
    cap = 4096
    arr = (c_u64 * cap)()
    r = c_int()
    _lib.call("nimbleMatrixFromText", text.encode(), arr, cap, ctypes.byref(r))
    return list(arr[: r.value * r.value]), r.value


# ------------------------------------------------------------------ planner

@dataclass
class CostModel:  # planner.hpp:36-49
    normalize_by_capacity: bool = True
    pi: float = 0.25
    small_message_cutoff: int = 1 * MiB
    saturation_intra: int = 64 * MiB
    saturation_inter: int = 32 * MiB

    @staticmethod
    def unpenalized():
        return CostModel(pi=0.0, small_message_cutoff=0)


@dataclass
class PlannerConfig:  # planner.hpp:51-56
    lam: float = 0.5
    epsilon: int = 4 * MiB
    cost: CostModel = field(default_factory=CostModel)
    max_pair_visits: int = 1_000_000

    def to_c(self) -> _lib.PlannerConfig:
        return _lib.PlannerConfig(self.lam, self.epsilon, self.cost.pi, self.cost.small_message_cutoff,
                                  self.cost.saturation_intra, self.cost.saturation_inter,
                                  self.max_pair_visits, int(self.cost.normalize_by_capacity))


@dataclass
class CandidatePath:  # planner.hpp:19-30
    cls: str
    via: int
    rail: int
    hops: int
    edges: list


@dataclass
class PairPlan:  # planner.hpp:63-69
    src: int
    dst: int
    demand: int
    candidates: list
    flows: list  # [(candidate index, bytes)]


@dataclass
class Plan:  # planner.hpp:80-84
    pairs: list
    stats: dict
    link_loads: list
    max_normalized_load: float
    json: str


def _read_plan(h, nlinks) -> Plan:
    L = _lib.lib()
    n = c_int()
    _lib.call("nimblePlanNumPairs", h, ctypes.byref(n))
    pairs = []
    for i in range(n.value):
        s, d, nc, nf = c_int(), c_int(), c_int(), c_int()
        dem = c_u64()
        _lib.call("nimblePlanPair", h, i, ctypes.byref(s), ctypes.byref(d), ctypes.byref(dem),
                  ctypes.byref(nc), ctypes.byref(nf))
        cands = []
        for c in range(nc.value):
            route, via, rail, hops, ne = c_int(), c_int(), c_int(), c_int(), c_int()
            edges = (c_int * 8)()
            _lib.call("nimblePlanCandidate", h, i, c, ctypes.byref(route), ctypes.byref(via),
                      ctypes.byref(rail), ctypes.byref(hops), edges, 8, ctypes.byref(ne))
            cands.append(CandidatePath(ROUTE_NAMES[route.value], via.value, rail.value, hops.value,
                                       list(edges[: ne.value])))
        flows = []
        for f in range(nf.value):
            cand, b = c_int(), c_double()
            _lib.call("nimblePlanFlow", h, i, f, ctypes.byref(cand), ctypes.byref(b))
            flows.append((cand.value, b.value))
        pairs.append(PairPlan(s.value, d.value, dem.value, cands, flows))
    st = _lib.PlanStats()
    _lib.call("nimblePlanGetStats", h, ctypes.byref(st))
    loads = (c_double * nlinks)()
    _lib.call("nimblePlanLinkLoads", h, loads, nlinks)
    mx = c_double()
    _lib.call("nimblePlanMaxNormalizedLoad", h, ctypes.byref(mx))
    need = c_size()
    L.nimblePlanToJson(h, None, 0, ctypes.byref(need))
    buf = ctypes.create_string_buffer(need.value)
    _lib.call("nimblePlanToJson", h, buf, need.value, ctypes.byref(need))
    stats = {k: getattr(st, k) for k, _ in _lib.PlanStats._fields_}
    return Plan(pairs, stats, list(loads), mx.value, buf.value.decode())


def _run(fn, topo: Topology, ranks, ranks_per_node, matrix, *extra) -> Plan:
    arr = _lib.u64_array(matrix)
    h = c_void_p()
    _lib.call(fn, topo.handle, ranks, ranks_per_node, arr, *extra, ctypes.byref(h))
    try:
        return _read_plan(h, topo.link_count())
    finally:
        _lib.lib().nimblePlanDestroy(h)


def plan(topo: Topology, ranks, ranks_per_node, matrix, config: PlannerConfig | None = None) -> Plan:
    """plan() -- planner.hpp:99-100."""
    cfg = (config or PlannerConfig()).to_c()
    return _run("nimblePlanCreate", topo, ranks, ranks_per_node, matrix, ctypes.byref(cfg))


def plan_direct_baseline(topo: Topology, ranks, ranks_per_node, matrix) -> Plan:
    """plan_direct_baseline() -- planner.hpp:103-104."""
    return _run("nimblePlanDirect", topo, ranks, ranks_per_node, matrix)


def enumerate_paths(topo: Topology, ranks, ranks_per_node, src, dst):
    """enumerate_paths() -- planner.hpp:86-87."""
    h = c_void_p()
    _lib.call("nimbleEnumeratePaths", topo.handle, ranks, ranks_per_node, src, dst, ctypes.byref(h))
    try:
        return _read_plan(h, topo.link_count()).pairs[0].candidates
    finally:
        _lib.lib().nimblePlanDestroy(h)


def plan_link_loads(p: Plan):
    return p.link_loads


def max_normalized_load(p: Plan):
    return p.max_normalized_load


def plan_to_json(p: Plan) -> dict:
    return json.loads(p.json)


def plan_from_json(topo: Topology, ranks, ranks_per_node, doc) -> Plan:
    """plan_from_json() -- planner.hpp:110 (accepts a dict or a JSON string)."""
    text = doc if isinstance(doc, str) else json.dumps(doc)
    h = c_void_p()
    _lib.call("nimblePlanFromJson", topo.handle, ranks, ranks_per_node, text.encode(), ctypes.byref(h))
    try:
        return _read_plan(h, topo.link_count())
    finally:
        _lib.lib().nimblePlanDestroy(h)


def port_bound_seconds(matrix, ranks, port_bytes_per_s=900e9):
    """The MCF roofline: max over GPUs of egress or ingress bytes / port rate."""
    worst = 0
    for v in range(ranks):
        worst = max(worst, sum(matrix[v * ranks:(v + 1) * ranks]),
                    sum(matrix[s * ranks + v] for s in range(ranks)))
    return worst / port_bytes_per_s


def debug_schedule(topo: Topology, ranks, ranks_per_node, matrix, rank, config: PlannerConfig | None = None,
                   pipe_chunk=64 * KiB, slots=160, direct_chunk=64 * KiB, staged_mask=0, pull_mask=0, push_chunk=0,
                   device=False):
    """The chunk scheduler's ordered work items for `rank` (nimbleDebugSchedule).

    push_chunk = 0 cuts direct pushes at direct_chunk.  device=True merges the
    flows with the GPU generator instead (nimbleDebugScheduleDevice; needs a
    GPU) -- the list must be the same.  Returns a list of
    dicts (kind, peer, aux, seq, src, dst, bytes).  The plan
    is mcf_plan on `topo` over the off-diagonal demands (self segments are
    plain local copies and are not part of it).
    """
    off_diag = [0 if i // ranks == i % ranks else v for i, v in enumerate(matrix)]
    cfg = (config or PlannerConfig()).to_c()
    h = c_void_p()
    _lib.call("nimblePlanCreate", topo.handle, ranks, ranks_per_node, _lib.u64_array(off_diag), ctypes.byref(cfg),
              ctypes.byref(h))
    try:
        n = c_int()
        fn = "nimbleDebugScheduleDevice" if device else "nimbleDebugSchedule"
        _lib.call(fn, h, rank, ranks, pipe_chunk, slots, direct_chunk, push_chunk, staged_mask, pull_mask,
                  None, 0, ctypes.byref(n))
        items = (_lib.Item * max(n.value, 1))()
        _lib.call(fn, h, rank, ranks, pipe_chunk, slots, direct_chunk, push_chunk, staged_mask, pull_mask,
                  items, n.value, ctypes.byref(n))
    finally:
        _lib.lib().nimblePlanDestroy(h)
    kinds = {0: "local", 1: "push", 2: "stage", 3: "forward", 4: "pull"}
    return [{"kind": kinds[it.kind], "peer": it.peer, "aux": it.aux, "seq": it.seq, "src": it.src, "dst": it.dst,
             "bytes": it.bytes} for it in items[:n.value]]
