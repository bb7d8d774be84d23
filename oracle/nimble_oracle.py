"""TEST INFRASTRUCTURE ONLY -- pure-Python restatement of the reference's
planning path (the parity oracle).

Restates, function by function, /root/reference/proj/src/{topology,workloads,
planner,pipeline}.cpp.  Python floats are IEEE-754 doubles and every load /
flow value on this path is an integer below 2**53, so the arithmetic is exact
and the restatement reproduces the reference bit for bit; the one long-double
product (gen_skewed_a2av) uses numpy.longdouble, the x87 80-bit type on
x86-64 Linux.  Pinned against the reference's own test vectors and against
oracle/_ref (tests/test_oracle_pins.py, tests/golden/).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product never does.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

KiB = 1024
MiB = 1024 * KiB
GiB = 1024 * MiB
INF = float("inf")


def gbps(x: float) -> float:  # proj/include/nimble/units.hpp:12
    return x * 1e9


# ---------------------------------------------------------------- topology
# proj/src/topology.cpp:70-179.  Link ids are dense, in construction order:
# intra-node links (mesh or switch ports), then attach pairs, then rails.

NVLINK, SWITCH_PORT, ATTACH, RAIL = 0, 1, 2, 3
ALLTOALL, NVSWITCH = "alltoall", "nvswitch"


@dataclass
class Topology:
    nodes: int
    gpus: int
    nics: int
    fabric: str
    nvlink_capacity: float
    rail_capacity: float
    kinds: list = field(default_factory=list)
    capacity: list = field(default_factory=list)
    ends: list = field(default_factory=list)  # (src, dst) device tuples

    def intra_per_node(self) -> int:  # topology.cpp:75-79
        return self.gpus * (self.gpus - 1) if self.fabric == ALLTOALL else 2 * self.gpus

    def nvlink_id(self, node, a, b):  # topology.cpp:83-89
        if self.fabric != ALLTOALL or a == b:
            raise LookupError("nvlink_id: no such link")
        return node * self.intra_per_node() + a * (self.gpus - 1) + (b if b < a else b - 1)

    def port_up_id(self, node, g):  # topology.cpp:91-94
        if self.fabric != NVSWITCH:
            raise LookupError("port_up_id: wrong fabric")
        return node * self.intra_per_node() + g

    def port_down_id(self, node, g):  # topology.cpp:96-99
        if self.fabric != NVSWITCH:
            raise LookupError("port_down_id: wrong fabric")
        return node * self.intra_per_node() + self.gpus + g

    def attach_up_id(self, node, nic):  # topology.cpp:101-104
        if nic < 0 or nic >= self.nics:
            raise LookupError("attach_up_id: bad nic")
        return self.nodes * self.intra_per_node() + node * 2 * self.nics + 2 * nic

    def attach_down_id(self, node, nic):  # topology.cpp:106-108
        return self.attach_up_id(node, nic) + 1

    def rail_id(self, a, b, r):  # topology.cpp:110-117
        if a == b or r < 0 or r >= self.nics:
            raise LookupError("rail_id: no such rail")
        base = self.nodes * self.intra_per_node() + self.nodes * 2 * self.nics
        return base + (a * (self.nodes - 1) + (b if b < a else b - 1)) * self.nics + r


def build_canonical(nodes, gpus, nics, nvlink_capacity, rail_capacity, fabric) -> Topology:
    """proj/src/topology.cpp:119-179."""
    if nodes < 1 or gpus < 1 or nics < 0 or nics > gpus or not nvlink_capacity > 0:
        raise ValueError("build_canonical: bad arguments")
    if nics > 0 and not rail_capacity > 0:
        raise ValueError("build_canonical: rail capacity must be positive")
    t = Topology(nodes, gpus, nics, fabric, nvlink_capacity, rail_capacity)

    def add(src, dst, kind, cap):
        t.ends.append((src, dst))
        t.kinds.append(kind)
        t.capacity.append(cap)

    for n in range(nodes):
        if fabric == ALLTOALL:
            for i in range(gpus):
                for j in range(gpus):
                    if i != j:
                        add(("g", n, i), ("g", n, j), NVLINK, nvlink_capacity)
        else:
            for i in range(gpus):
                add(("g", n, i), ("sw", n, 0), SWITCH_PORT, nvlink_capacity)
            for i in range(gpus):
                add(("sw", n, 0), ("g", n, i), SWITCH_PORT, nvlink_capacity)
    for n in range(nodes):
        for k in range(nics):
            add(("g", n, k), ("nic", n, k), ATTACH, 2 * rail_capacity)
            add(("nic", n, k), ("g", n, k), ATTACH, 2 * rail_capacity)
    for a in range(nodes):
        for b in range(nodes):
            if a != b:
                for r in range(nics):
                    add(("nic", a, r), ("nic", b, r), RAIL, rail_capacity)
    return t


# ---------------------------------------------------------------- workloads
# proj/src/workloads.cpp.  Matrices are flat row-major lists, row = sender.

def _blank(ranks):
    if ranks < 2:
        raise ValueError("workload: need at least 2 ranks")
    return [0] * (ranks * ranks)


def gen_p2p(ranks, src, dst, size):  # workloads.cpp:46-53
    m = _blank(ranks)
    if not (0 <= src < ranks and 0 <= dst < ranks) or src == dst:
        raise ValueError("p2p: bad ranks")
    m[src * ranks + dst] = size
    return m


def _split_even(total, peers, m, ranks, sender):  # workloads.cpp:57-64
    if not peers:
        return
    base, rem = divmod(total, len(peers))
    for i, p in enumerate(peers):
        m[sender * ranks + p] = base + (rem if i + 1 == len(peers) else 0)


def gen_skewed_a2av(ranks, per_rank, ratio, hot=0, seed=0, per_sender_hot=False):
    """workloads.cpp:66-92; the hot share is floor(ratio * P) in long double."""
    m = _blank(ranks)
    if not 0 <= hot < ranks:
        raise ValueError("skewed: hot_dst out of range")
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("skewed: ratio must be in [0,1]")
    for s in range(ranks):
        h = hot
        if per_sender_hot:
            h = (hot + s) % ranks
            if h == s:
                h = (h + 1) % ranks
        cold = [d for d in range(ranks) if d != s and d != h]
        if s == h:
            _split_even(per_rank, cold, m, ranks, s)
            continue
        share = int(np.floor(np.longdouble(ratio) * np.longdouble(per_rank)))
        m[s * ranks + h] = share
        _split_even(per_rank - share, cold, m, ranks, s)
    return m


def gen_stencil_1d(ranks, halo):  # workloads.cpp:94-101
    m = _blank(ranks)
    for r in range(ranks - 1):
        m[r * ranks + r + 1] = halo
        m[(r + 1) * ranks + r] = halo
    return m


def gen_aggregator(ranks, dsts, per_src):  # workloads.cpp:103-115
    m = _blank(ranks)
    dsts = sorted(set(dsts))
    if not dsts or any(d < 0 or d >= ranks for d in dsts):
        raise ValueError("aggregator: bad destination set")
    for s in range(ranks):
        if s not in dsts:
            _split_even(per_src, dsts, m, ranks, s)
    return m


class MT19937_64:
    """std::mt19937_64 (the standard fully specifies its output)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) \
                & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def __call__(self):
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def gen_irregular(ranks, total, sparsity, seed):  # workloads.cpp:117-152
    if not (0.0 < sparsity <= 1.0):
        raise ValueError("irregular: sparsity must be in (0,1]")
    m = _blank(ranks)
    rng = MT19937_64(seed)

    def u01():
        return float(rng() >> 11) * 2.0 ** -53

    kept = []
    for s in range(ranks):
        for d in range(ranks):
            if s != d and u01() < sparsity:
                kept.append(s * ranks + d)
    if not kept:
        kept.append(1)
    w = []
    wsum = 0.0
    for _ in kept:
        x = u01() + 1e-9
        w.append(x)
        wsum += x
    assigned = 0
    for i, k in enumerate(kept):
        v = int(math.floor(float(total) * w[i] / wsum))
        m[k] = v
        assigned += v
    left = total - assigned
    i = 0
    while left > 0:
        m[kept[i]] += 1
        i = (i + 1) % len(kept)
        left -= 1
    return m


def write_payload_matrix(m, ranks):  # workloads.cpp:154-164
    return "".join(" ".join(str(m[s * ranks + d]) for d in range(ranks)) + "\n"
                   for s in range(ranks))


# ---------------------------------------------------------------- planner
# proj/src/planner.cpp

DIRECT, TWO_HOP, INTER_RAIL = "direct", "intra_two_hop", "inter_rail"


@dataclass
class Candidate:
    cls: str
    via: int = -1
    rail: int = -1
    hops: int = 1
    pair_direct: bool = False
    edges: list = field(default_factory=list)


@dataclass
class CostModel:  # planner.hpp:36-49
    normalize: bool = True
    pi: float = 0.25
    small_message_cutoff: int = 1 * MiB
    saturation_intra: int = 64 * MiB
    saturation_inter: int = 32 * MiB

    def hop_penalty(self, c: Candidate, message: int) -> float:  # planner.cpp:12-19
        if c.hops <= 1:
            return 0.0
        if message <= self.small_message_cutoff:
            return INF
        sat = self.saturation_inter if c.cls == INTER_RAIL else self.saturation_intra
        fade = 1.0 - float(message) / float(sat)
        if fade <= 0.0:
            return 0.0
        return self.pi * float(c.hops - 1) * fade

    @staticmethod
    def unpenalized():  # planner.cpp:21-26
        return CostModel(pi=0.0, small_message_cutoff=0)


@dataclass
class PlannerConfig:  # planner.hpp:51-56
    lam: float = 0.5
    epsilon: int = 4 * MiB
    cost: CostModel = field(default_factory=CostModel)
    max_pair_visits: int = 1_000_000


def _intra_edges(t: Topology, node, a, b, out):  # planner.cpp:28-37
    if a == b:
        return
    if t.fabric == ALLTOALL:
        out.append(t.nvlink_id(node, a, b))
    else:
        out.append(t.port_up_id(node, a))
        out.append(t.port_down_id(node, b))


def enumerate_paths(t: Topology, ranks, rpn, s, d):
    """planner.cpp:39-108."""
    if not (0 <= s < ranks and 0 <= d < ranks):
        raise ValueError("enumerate_paths: rank out of range")
    if s == d:
        raise ValueError("enumerate_paths: src equals dst")
    sn, so, dn, dd = s // rpn, s % rpn, d // rpn, d % rpn
    if sn >= t.nodes or dn >= t.nodes or so >= t.gpus or dd >= t.gpus:
        raise ValueError("enumerate_paths: rank map exceeds topology")
    out = []
    if sn == dn:
        c = Candidate(DIRECT, hops=1, pair_direct=True)
        _intra_edges(t, sn, so, dd, c.edges)
        out.append(c)
        if t.fabric == ALLTOALL:
            for v in range(t.gpus):
                if v in (so, dd):
                    continue
                out.append(Candidate(TWO_HOP, via=v, hops=2,
                                     edges=[t.nvlink_id(sn, so, v), t.nvlink_id(sn, v, dd)]))
        return out
    if t.nics == 0:
        raise ValueError("enumerate_paths: no rails between nodes")

    def rail(r):
        c = Candidate(INTER_RAIL, rail=r, hops=1 + (so != r) + (dd != r))
        _intra_edges(t, sn, so, r, c.edges)
        c.edges += [t.attach_up_id(sn, r), t.rail_id(sn, dn, r), t.attach_down_id(dn, r)]
        _intra_edges(t, dn, r, dd, c.edges)
        return c

    direct_rail = dd % t.nics
    c = rail(direct_rail)
    c.pair_direct = True
    c.hops = 1
    out.append(c)
    out += [rail(r) for r in range(t.nics) if r != direct_rail]
    return out


def path_cost(c: Candidate, loads, t: Topology, cost: CostModel, message, pending=0.0):
    """planner.cpp:110-120."""
    worst = 0.0
    for e in c.edges:
        v = (loads[e] + pending) / t.capacity[e] if cost.normalize else loads[e] + pending
        worst = max(worst, v)
    return worst + cost.hop_penalty(c, message)


@dataclass
class PairPlan:
    src: int
    dst: int
    demand: int
    candidates: list
    flows: list = field(default_factory=list)  # (candidate index, bytes)


@dataclass
class Plan:
    pairs: list
    epsilon: int = 4 * MiB
    stats: dict = field(default_factory=dict)


def _pairs(t, ranks, rpn, m):  # planner.cpp:302-318
    out = []
    for s in range(ranks):
        for d in range(ranks):
            if s == d:
                if m[s * ranks + d]:
                    raise ValueError("demand matrix: nonzero diagonal")
                continue
            if m[s * ranks + d]:
                out.append(PairPlan(s, d, m[s * ranks + d], enumerate_paths(t, ranks, rpn, s, d)))
    return out


def _global_max(t, loads):
    w = 0.0
    for e, l in enumerate(loads):
        w = max(w, l / t.capacity[e])
    return w


def _refine(t: Topology, pairs, acc, loads, cfg: PlannerConfig):
    """planner.cpp:131-300: reduce / consolidate / eject passes, 8 rounds."""
    MOVE_CAP, EJECT_TRIES = 4096, 4096
    eps = float(cfg.epsilon)
    st = {"moves": 0, "eject": 0}

    def norm(e):
        return loads[e] / t.capacity[e]

    def shift(i, a, b, q):
        for e in pairs[i].candidates[a].edges:
            loads[e] -= q
        for e in pairs[i].candidates[b].edges:
            loads[e] += q
        acc[i][a] -= q
        acc[i][b] += q

    def pen(i, c):
        return cfg.cost.hop_penalty(pairs[i].candidates[c], pairs[i].demand)

    def reduce_pass():
        any_ = False
        progress = True
        while progress and st["moves"] < MOVE_CAP:
            progress = False
            cur = _global_max(t, loads)
            if cur <= 0.0:
                break
            bar = cur * (1.0 - 1e-12)
            for i in range(len(pairs)):
                if progress:
                    break
                cands = pairs[i].candidates
                for c in range(len(cands)):
                    if progress:
                        break
                    if acc[i][c] <= 0.0:
                        continue
                    if not any(norm(e) >= bar for e in cands[c].edges):
                        continue
                    q = min(eps, acc[i][c])
                    p = pen(i, c)
                    for a in range(len(cands)):
                        if a == c or pen(i, a) > p:
                            continue
                        shift(i, c, a, q)
                        if _global_max(t, loads) < bar:
                            st["moves"] += 1
                            progress = any_ = True
                            break
                        shift(i, a, c, q)
        return any_

    def consolidate_pass():
        any_ = False
        progress = True
        while progress and st["moves"] < MOVE_CAP:
            progress = False
            cur = _global_max(t, loads)
            bar = cur * (1.0 - 1e-12)
            for i in range(len(pairs)):
                cands = pairs[i].candidates
                for c in range(1, len(cands)):
                    while acc[i][c] > 0.0 and st["moves"] < MOVE_CAP:
                        q = min(eps, acc[i][c])
                        shift(i, c, 0, q)
                        if any(norm(e) >= bar for e in cands[0].edges):
                            shift(i, 0, c, q)
                            break
                        st["moves"] += 1
                        progress = any_ = True
                        nm = _global_max(t, loads)
                        if nm < cur:
                            cur = nm
                            bar = cur * (1.0 - 1e-12)
        return any_

    def eject_pass():
        if st["moves"] + 2 > MOVE_CAP:
            return False
        cur = _global_max(t, loads)
        if cur <= 0.0:
            return False
        bar = cur * (1.0 - 1e-12)
        for i in range(len(pairs)):
            cands = pairs[i].candidates
            for c in range(len(cands)):
                if acc[i][c] <= 0.0:
                    continue
                if not any(norm(e) >= bar for e in cands[c].edges):
                    continue
                q = min(eps, acc[i][c])
                p = pen(i, c)
                for a in range(len(cands)):
                    if a == c or pen(i, a) > p:
                        continue
                    shift(i, c, a, q)
                    for be in cands[a].edges:
                        if norm(be) < bar:
                            continue
                        for j in range(len(pairs)):
                            jc = pairs[j].candidates
                            for d in range(len(jc)):
                                if j == i and (d == a or d == c):
                                    continue
                                if acc[j][d] <= 0.0:
                                    continue
                                if be not in jc[d].edges:
                                    continue
                                v = min(eps, acc[j][d])
                                jp = pen(j, d)
                                for b in range(len(jc)):
                                    if b == d or pen(j, b) > jp:
                                        continue
                                    if st["eject"] >= EJECT_TRIES:
                                        break
                                    st["eject"] += 1
                                    shift(j, d, b, v)
                                    if _global_max(t, loads) < bar:
                                        st["moves"] += 2
                                        return True
                                    shift(j, b, d, v)
                    shift(i, a, c, q)
                    if st["eject"] >= EJECT_TRIES:
                        return False
        return False

    for _ in range(8):
        r = reduce_pass()
        c = consolidate_pass()
        if not r and not c and not eject_pass():
            break
    return st["moves"]


def plan(t: Topology, ranks, rpn, m, cfg: PlannerConfig | None = None) -> Plan:
    """planner.cpp:320-429: lambda/epsilon sweep, refinement, direct guard."""
    cfg = cfg or PlannerConfig()
    if not (0.0 < cfg.lam <= 1.0):
        raise ValueError("planner: lambda must be in (0,1]")
    if cfg.epsilon == 0:
        raise ValueError("planner: epsilon must be positive")
    pairs = _pairs(t, ranks, rpn, m)
    stats = dict(pair_visits=0, placements=0, fallback_pairs=0, residual_flows=0, refine_moves=0)
    loads = [0.0] * len(t.capacity)
    acc = [[0.0] * len(p.candidates) for p in pairs]
    remaining = [float(p.demand) for p in pairs]
    active = list(range(len(pairs)))
    eps = float(cfg.epsilon)
    out_of_visits = False
    while active and not out_of_visits:
        still = []
        for i in active:
            if stats["pair_visits"] >= cfg.max_pair_visits:
                out_of_visits = True
                still.append(i)
                continue
            stats["pair_visits"] += 1
            pp = pairs[i]
            r = remaining[i]
            budget = r if r < eps else max(eps, math.floor(r * cfg.lam / eps) * eps)
            while budget > 0.0:
                chunk = min(eps, budget)
                best, best_cost = 0, INF
                for c, cand in enumerate(pp.candidates):
                    pc = path_cost(cand, loads, t, cfg.cost, pp.demand, chunk)
                    if pc < best_cost:
                        best, best_cost = c, pc
                for e in pp.candidates[best].edges:
                    loads[e] += chunk
                acc[i][best] += chunk
                stats["placements"] += 1
                if chunk < eps:
                    stats["residual_flows"] += 1
                budget -= chunk
                r -= chunk
            remaining[i] = r
            if r > 0.0:
                still.append(i)
        active = still
    if out_of_visits:
        for i in active:
            acc[i][0] += remaining[i]
            for e in pairs[i].candidates[0].edges:
                loads[e] += remaining[i]
            stats["fallback_pairs"] += 1
    stats["refine_moves"] = _refine(t, pairs, acc, loads, cfg)
    direct = [0.0] * len(t.capacity)
    for p in pairs:
        for e in p.candidates[0].edges:
            direct[e] += float(p.demand)
    if _global_max(t, loads) > _global_max(t, direct) * (1.0 + 1e-12):
        for i, p in enumerate(pairs):
            acc[i] = [0.0] * len(p.candidates)
            acc[i][0] = float(p.demand)
        loads[:] = direct
        stats["refine_moves"] += _refine(t, pairs, acc, loads, cfg)
    for i, p in enumerate(pairs):
        p.flows = [(c, b) for c, b in enumerate(acc[i]) if b > 0.0]
    return Plan(pairs, cfg.epsilon, stats)


def plan_direct_baseline(t, ranks, rpn, m) -> Plan:  # planner.cpp:431-438
    pairs = _pairs(t, ranks, rpn, m)
    for p in pairs:
        p.flows = [(0, float(p.demand))]
    return Plan(pairs, 4 * MiB, {})


def plan_link_loads(t, p: Plan):  # planner.cpp:440-447
    loads = [0.0] * len(t.capacity)
    for pp in p.pairs:
        for c, b in pp.flows:
            for e in pp.candidates[c].edges:
                loads[e] += b
    return loads


def max_normalized_load(t, p: Plan):  # planner.cpp:449-455
    return _global_max(t, plan_link_loads(t, p))


def port_bound_seconds(m, ranks, port_bytes_per_s):
    """MCF port bound of SURVEY.md sec. 8(d): max over GPUs of egress/ingress bytes
    over the port rate; equals max_normalized_load of the direct plan on the
    nvswitch model."""
    worst = 0
    for v in range(ranks):
        eg = sum(m[v * ranks + d] for d in range(ranks))
        ig = sum(m[s * ranks + v] for s in range(ranks))
        worst = max(worst, eg, ig)
    return worst / port_bytes_per_s


# ---------------------------------------------------------------- pipeline
# proj/src/pipeline.cpp:29-32 and :66-116 -- the flow-control recurrence the
# forwarding engine's ready / consumed flags implement.

def slots(p2p_buffer=10 * MiB, pipe_chunk=512 * KiB, channels=1):
    return 0 if pipe_chunk == 0 else channels * (p2p_buffer // pipe_chunk)


def chunk_sizes(message, pipe_chunk):
    """pipeline.cpp:85-91: ceil(m / c) chunks, the last one short."""
    if message == 0:
        return []
    n = -(-message // pipe_chunk)
    return [pipe_chunk] * (n - 1) + [message - pipe_chunk * (n - 1)]


def simulate_transfer(chain, message, pipe_chunk=512 * KiB, p2p_buffer=10 * MiB, channels=1):
    """pipeline.cpp:97-106: start[h][k] = max(delivered[h-1][k], tx_done[h][k-1],
    tx_done[h+1][k-S]).  Returns (completion, start, tx_done, delivered)."""
    S = slots(p2p_buffer, pipe_chunk, channels)
    sizes = [float(x) for x in chunk_sizes(int(message), pipe_chunk)]
    n, H = len(sizes), len(chain)
    start = [[0.0] * n for _ in range(H)]
    txd = [[0.0] * n for _ in range(H)]
    dlv = [[0.0] * n for _ in range(H)]
    for k in range(n):
        for h in range(H):
            t = 0.0 if h == 0 else dlv[h - 1][k]
            if k > 0:
                t = max(t, txd[h][k - 1])
            if h + 1 < H and k >= S:
                t = max(t, txd[h + 1][k - S])
            start[h][k] = t
            txd[h][k] = t + sizes[k] / chain[h][0]
            dlv[h][k] = txd[h][k] + chain[h][1]
    return (dlv[H - 1][n - 1] if n else 0.0), start, txd, dlv
