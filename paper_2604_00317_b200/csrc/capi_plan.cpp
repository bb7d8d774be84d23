#include <cuda_runtime.h>
// C ABI, group 1: link-load model, traffic-matrix ingest, planner.
// Host-only; exceptions from the C++ core become result codes here.
#include <algorithm>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/nimble.h"
#include "capi_util.hpp"
#include "demand.hpp"
#include "fabric.hpp"
#include "planner.hpp"
#include "device.cuh"
#include "schedule.hpp"

struct nimbleTopology {
    nb::LinkModel lm;
};

struct nimblePlan {
    nb::LinkModel lm;
    nb::PlanResult plan;
};

namespace nb {

thread_local std::string g_last_error;

nimbleResult_t fail(nimbleResult_t code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

nimbleResult_t write_text(const std::string& s, char* out, size_t cap, size_t* need) {
    if (need) *need = s.size() + 1;
    if (!out || cap < s.size() + 1) return fail(nimbleInvalidArgument, "output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
    return nimbleSuccess;
}

PlanParams to_params(const nimblePlannerConfig* c) {
    PlanParams p;
    if (!c) return p;
    p.lambda = c->lambda;
    p.epsilon = c->epsilon;
    p.cost.pi = c->pi;
    p.cost.cutoff = c->small_message_cutoff;
    p.cost.sat_intra = c->saturation_intra;
    p.cost.sat_inter = c->saturation_inter;
    p.cost.normalize = c->normalize_by_capacity != 0;
    p.max_visits = c->max_pair_visits;
    return p;
}

Demand to_demand(int ranks, const uint64_t* m) {
    if (ranks < 1 || !m) throw std::invalid_argument("matrix: need ranks >= 1 and a matrix");
    Demand d;
    d.ranks = ranks;
    d.bytes.assign(m, m + static_cast<size_t>(ranks) * ranks);
    d.check();
    return d;
}

}  // namespace nb

using nb::fail;

extern "C" {

const char* nimbleGetErrorString(nimbleResult_t r) {
    switch (r) {
    case nimbleSuccess: return "no error";
    case nimbleUnhandledCudaError: return "unhandled cuda error";
    case nimbleSystemError: return "unhandled system error";
    case nimbleInternalError: return "internal error";
    case nimbleInvalidArgument: return "invalid argument";
    case nimbleInvalidUsage: return "invalid usage";
    case nimbleRemoteError: return "remote process exited or there was a network error";
    case nimbleInProgress: return "operation in progress";
    default: return "unknown result code";
    }
}

const char* nimbleGetLastError(void) { return nb::g_last_error.c_str(); }

nimbleResult_t nimbleGetVersion(int* v) {
    if (!v) return fail(nimbleInvalidArgument, "version: null pointer");
    *v = NIMBLE_VERSION_CODE;
    return nimbleSuccess;
}

nimbleResult_t nimbleTopologyCreate(int nodes, int gpus, int nics, double nv, double rail,
                                    nimbleFabric_t fabric, nimbleTopology_t* out) {
    return nb::guarded([&] {
        if (!out) throw std::invalid_argument("topology: null output");
        auto* t = new nimbleTopology{nb::make_link_model(
            nodes, gpus, nics, nv, rail,
            fabric == nimbleFabricAllToAll ? nb::FabricKind::AllToAll : nb::FabricKind::NvSwitch)};
        *out = t;
    });
}

nimbleResult_t nimbleTopologyLoad(const char* text, nimbleTopology_t* out) {
    return nb::guarded([&] {
        if (!text || !out) throw std::invalid_argument("topology: null argument");
        *out = new nimbleTopology{nb::load_link_model(text)};
    });
}

nimbleResult_t nimbleTopologySave(nimbleTopology_t t, char* out, size_t cap, size_t* need) {
    if (!t) return fail(nimbleInvalidArgument, "topology: null handle");
    return nb::write_text(nb::save_link_model(t->lm), out, cap, need);
}

nimbleResult_t nimbleTopologyDestroy(nimbleTopology_t t) {
    delete t;
    return nimbleSuccess;
}

nimbleResult_t nimbleTopologyLinkCount(nimbleTopology_t t, int* n) {
    if (!t || !n) return fail(nimbleInvalidArgument, "topology: null argument");
    *n = t->lm.links();
    return nimbleSuccess;
}

nimbleResult_t nimbleTopologyLink(nimbleTopology_t t, int id, int* kind, double* cap, char* name,
                                  size_t name_cap) {
    if (!t || id < 0 || id >= t->lm.links()) return fail(nimbleInvalidArgument, "topology: bad link id");
    if (kind) *kind = static_cast<int>(t->lm.cls[id]);
    if (cap) *cap = t->lm.cap[id];
    if (name && name_cap) {
        std::string s = t->lm.name(id);
        std::strncpy(name, s.c_str(), name_cap - 1);
        name[name_cap - 1] = 0;
    }
    return nimbleSuccess;
}

nimbleResult_t nimbleTopologySetCapacity(nimbleTopology_t t, int id, double bw) {
    if (!t || id < 0 || id >= t->lm.links() || !(bw > 0))
        return fail(nimbleInvalidArgument, "topology: bad link id or capacity");
    t->lm.cap[id] = bw;
    return nimbleSuccess;
}

nimbleResult_t nimbleTopologyLinkId(nimbleTopology_t t, int kind, int node, int a, int b, int* id) {
    return nb::guarded([&] {
        if (!t || !id) throw std::invalid_argument("topology: null argument");
        *id = -1;
        switch (kind) {
        case nimbleLinkNvLink: *id = t->lm.mesh(node, a, b); break;
        case nimbleLinkSwitchPort: *id = b ? t->lm.down(node, a) : t->lm.up(node, a); break;
        case nimbleLinkAttach: *id = b ? t->lm.attach_down(node, a) : t->lm.attach_up(node, a); break;
        case nimbleLinkRail: *id = t->lm.rail(node, a, b); break;
        default: throw std::invalid_argument("topology: bad link kind");
        }
    });
}

static void emit(const nb::Demand& d, uint64_t* out) {
    if (!out) throw std::invalid_argument("matrix: null output");
    std::memcpy(out, d.bytes.data(), d.bytes.size() * sizeof(uint64_t));
}

nimbleResult_t nimbleGenP2P(int ranks, int src, int dst, uint64_t size, uint64_t* m) {
    return nb::guarded([&] { emit(nb::demand_p2p(ranks, src, dst, size), m); });
}

nimbleResult_t nimbleGenSkewed(int ranks, uint64_t per_rank, double ratio, int hot, int psh, uint64_t* m) {
    return nb::guarded([&] { emit(nb::demand_skewed(ranks, per_rank, ratio, hot, psh != 0), m); });
}

nimbleResult_t nimbleGenStencil1D(int ranks, uint64_t halo, uint64_t* m) {
    return nb::guarded([&] { emit(nb::demand_stencil(ranks, halo), m); });
}

nimbleResult_t nimbleGenAggregator(int ranks, const int* dsts, int n, uint64_t per_src, uint64_t* m) {
    return nb::guarded([&] {
        std::vector<int> v;
        if (n > 0 && dsts) v.assign(dsts, dsts + n);
        emit(nb::demand_aggregator(ranks, v, per_src), m);
    });
}

nimbleResult_t nimbleGenIrregular(int ranks, uint64_t total, double sparsity, uint64_t seed, uint64_t* m) {
    return nb::guarded([&] { emit(nb::demand_irregular(ranks, total, sparsity, seed), m); });
}

nimbleResult_t nimbleMatrixToText(int ranks, const uint64_t* m, char* out, size_t cap, size_t* need) {
    std::string s;
    nimbleResult_t r = nb::guarded([&] { s = nb::demand_to_text(nb::to_demand(ranks, m)); });
    if (r != nimbleSuccess) return r;
    return nb::write_text(s, out, cap, need);
}

nimbleResult_t nimbleMatrixFromText(const char* text, uint64_t* m, size_t cap, int* ranks) {
    return nb::guarded([&] {
        if (!text || !ranks) throw std::invalid_argument("matrix: null argument");
        nb::Demand d = nb::demand_from_text(text);
        *ranks = d.ranks;
        if (!m || cap < d.bytes.size()) throw std::invalid_argument("matrix: output too small");
        std::memcpy(m, d.bytes.data(), d.bytes.size() * sizeof(uint64_t));
    });
}

nimbleResult_t nimblePlannerConfigDefault(nimblePlannerConfig* c) {
    if (!c) return fail(nimbleInvalidArgument, "planner config: null");
    nb::PlanParams p;
    c->lambda = p.lambda;
    c->epsilon = p.epsilon;
    c->pi = p.cost.pi;
    c->small_message_cutoff = p.cost.cutoff;
    c->saturation_intra = p.cost.sat_intra;
    c->saturation_inter = p.cost.sat_inter;
    c->max_pair_visits = p.max_visits;
    c->normalize_by_capacity = 1;
    return nimbleSuccess;
}

nimbleResult_t nimblePlanCreate(nimbleTopology_t t, int ranks, int rpn, const uint64_t* m,
                                const nimblePlannerConfig* cfg, nimblePlan_t* out) {
    return nb::guarded([&] {
        if (!t || !out) throw std::invalid_argument("plan: null argument");
        auto* p = new nimblePlan{t->lm, {}};
        try {
            p->plan = nb::mcf_plan(t->lm, ranks, rpn, nb::to_demand(ranks, m), nb::to_params(cfg));
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

nimbleResult_t nimblePlanDirect(nimbleTopology_t t, int ranks, int rpn, const uint64_t* m, nimblePlan_t* out) {
    return nb::guarded([&] {
        if (!t || !out) throw std::invalid_argument("plan: null argument");
        auto* p = new nimblePlan{t->lm, {}};
        try {
            p->plan = nb::direct_plan(t->lm, ranks, rpn, nb::to_demand(ranks, m));
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

nimbleResult_t nimbleEnumeratePaths(nimbleTopology_t t, int ranks, int rpn, int src, int dst, nimblePlan_t* out) {
    return nb::guarded([&] {
        if (!t || !out) throw std::invalid_argument("enumerate_paths: null argument");
        auto* p = new nimblePlan{t->lm, {}};
        try {
            nb::PairRoutes pr;
            pr.src = src;
            pr.dst = dst;
            pr.cands = nb::routes_for(t->lm, ranks, rpn, src, dst);
            p->plan.pairs.push_back(std::move(pr));
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

nimbleResult_t nimblePlanFromJson(nimbleTopology_t t, int ranks, int rpn, const char* json, nimblePlan_t* out) {
    return nb::guarded([&] {
        if (!t || !json || !out) throw std::invalid_argument("plan json: null argument");
        auto* p = new nimblePlan{t->lm, {}};
        try {
            p->plan = nb::plan_from_json(t->lm, ranks, rpn, json);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

nimbleResult_t nimblePlanDestroy(nimblePlan_t p) {
    delete p;
    return nimbleSuccess;
}

nimbleResult_t nimblePlanNumPairs(nimblePlan_t p, int* n) {
    if (!p || !n) return fail(nimbleInvalidArgument, "plan: null argument");
    *n = static_cast<int>(p->plan.pairs.size());
    return nimbleSuccess;
}

nimbleResult_t nimblePlanPair(nimblePlan_t p, int i, int* src, int* dst, uint64_t* demand, int* nc, int* nf) {
    if (!p || i < 0 || i >= static_cast<int>(p->plan.pairs.size()))
        return fail(nimbleInvalidArgument, "plan: bad pair index");
    const nb::PairRoutes& pr = p->plan.pairs[static_cast<size_t>(i)];
    if (src) *src = pr.src;
    if (dst) *dst = pr.dst;
    if (demand) *demand = pr.demand;
    if (nc) *nc = static_cast<int>(pr.cands.size());
    if (nf) *nf = static_cast<int>(pr.flows.size());
    return nimbleSuccess;
}

nimbleResult_t nimblePlanCandidate(nimblePlan_t p, int i, int c, int* route, int* via, int* rail,
                                   int* hops, int* edges, int cap, int* ne) {
    if (!p || i < 0 || i >= static_cast<int>(p->plan.pairs.size()))
        return fail(nimbleInvalidArgument, "plan: bad pair index");
    const nb::PairRoutes& pr = p->plan.pairs[static_cast<size_t>(i)];
    if (c < 0 || c >= static_cast<int>(pr.cands.size())) return fail(nimbleInvalidArgument, "plan: bad candidate");
    const nb::Candidate& k = pr.cands[static_cast<size_t>(c)];
    if (route) *route = static_cast<int>(k.route);
    if (via) *via = k.via;
    if (rail) *rail = k.rail;
    if (hops) *hops = k.hops;
    if (ne) *ne = k.ne;
    if (edges)
        for (int e = 0; e < k.ne && e < cap; ++e) edges[e] = k.e[e];
    return nimbleSuccess;
}

nimbleResult_t nimblePlanFlow(nimblePlan_t p, int i, int f, int* cand, double* bytes) {
    if (!p || i < 0 || i >= static_cast<int>(p->plan.pairs.size()))
        return fail(nimbleInvalidArgument, "plan: bad pair index");
    const nb::PairRoutes& pr = p->plan.pairs[static_cast<size_t>(i)];
    if (f < 0 || f >= static_cast<int>(pr.flows.size())) return fail(nimbleInvalidArgument, "plan: bad flow");
    if (cand) *cand = pr.flows[static_cast<size_t>(f)].cand;
    if (bytes) *bytes = pr.flows[static_cast<size_t>(f)].bytes;
    return nimbleSuccess;
}

nimbleResult_t nimblePlanGetStats(nimblePlan_t p, nimblePlanStats* s) {
    if (!p || !s) return fail(nimbleInvalidArgument, "plan: null argument");
    const nb::PlanCounters& c = p->plan.stats;
    *s = {c.pair_visits, c.placements, c.fallback_pairs, c.residual_flows, c.refine_moves, c.wall_seconds};
    return nimbleSuccess;
}

nimbleResult_t nimblePlanLinkLoads(nimblePlan_t p, double* loads, int n) {
    if (!p || !loads || n < p->lm.links()) return fail(nimbleInvalidArgument, "plan: loads buffer too small");
    const std::vector<double> l = nb::link_loads(p->lm, p->plan);
    std::memcpy(loads, l.data(), l.size() * sizeof(double));
    return nimbleSuccess;
}

nimbleResult_t nimblePlanMaxNormalizedLoad(nimblePlan_t p, double* s) {
    if (!p || !s) return fail(nimbleInvalidArgument, "plan: null argument");
    *s = nb::peak_load(p->lm, p->plan);
    return nimbleSuccess;
}

nimbleResult_t nimblePlanToJson(nimblePlan_t p, char* out, size_t cap, size_t* need) {
    if (!p) return fail(nimbleInvalidArgument, "plan: null handle");
    return nb::write_text(nb::plan_json(p->plan), out, cap, need);
}

}  // extern "C"

namespace nb {
cudaError_t launch_gen(const GenArgs& g, cudaStream_t st);
namespace {

// nimbleDebugSchedule's rank buffers: synthetic addresses, packed layout.
Schedule debug_schedule(nimblePlan_t p, int rank, int ranks, uint64_t pipe_chunk, uint32_t slots,
                        uint64_t direct_chunk, uint64_t push_chunk, uint64_t staged, uint64_t pull) {
    if (!p || ranks < 1 || ranks > kMaxRanks || rank < 0 || rank >= ranks)
        throw std::invalid_argument("schedule: bad argument");
    std::vector<uint64_t> m(static_cast<size_t>(ranks) * ranks, 0);
    for (const PairRoutes& pr : p->plan.pairs) m[static_cast<size_t>(pr.src) * ranks + pr.dst] = pr.demand;
    RankBuffers rb;
    rb.R = ranks;
    rb.me = rank;
    rb.send_ptr.assign(ranks, 0);
    rb.send_bytes.assign(ranks, 0);
    rb.recv_ptr.assign(ranks, 0);
    rb.recv_bytes.assign(ranks, 0);
    rb.recv_post.assign(ranks, Post{});
    rb.send_post.assign(ranks, Post{});
    uint64_t so = 0, ro = 0;
    for (int q = 0; q < ranks; ++q) {
        rb.send_bytes[q] = m[static_cast<size_t>(rank) * ranks + q];
        rb.send_ptr[q] = (static_cast<uint64_t>(1 + rank) << 40) + so;
        so += rb.send_bytes[q];
        rb.recv_bytes[q] = m[static_cast<size_t>(q) * ranks + rank];
        rb.recv_ptr[q] = (static_cast<uint64_t>(17 + rank) << 40) + ro;
        ro += rb.recv_bytes[q];
        if (q != rank && rb.recv_bytes[q]) {
            Post& post = rb.recv_post[q];
            post.tag = 1;
            post.bytes = rb.recv_bytes[q];
            post.mode = ((staged >> q) & 1) ? kPostStaged : kPostZeroCopy;
            if ((pull >> q) & 1) post.mode |= kPostPullRequest;
        }
    }
    return build_schedule(p->plan, rb, pipe_chunk, slots, direct_chunk, push_chunk);
}

}  // namespace
}  // namespace nb

extern "C" {

nimbleResult_t nimbleDebugSchedule(nimblePlan_t p, int rank, int ranks, uint64_t pipe_chunk, uint32_t slots,
                                   uint64_t direct_chunk, uint64_t push_chunk, uint64_t staged, uint64_t pull,
                                   nimbleItem* items, int cap, int* nitems) {
    static_assert(sizeof(nimbleItem) == sizeof(nb::Item), "nimbleItem mirrors the engine's Item");
    return nb::guarded([&] {
        if (!nitems) throw std::invalid_argument("schedule: bad argument");
        nb::Schedule sc = nb::debug_schedule(p, rank, ranks, pipe_chunk, slots, direct_chunk, push_chunk, staged, pull);
        nb::materialize(sc);
        *nitems = static_cast<int>(sc.items.size());
        if (items) std::memcpy(items, sc.items.data(), std::min<size_t>(sc.items.size(), cap > 0 ? cap : 0) * sizeof(nb::Item));
    });
}

nimbleResult_t nimbleDebugScheduleDevice(nimblePlan_t p, int rank, int ranks, uint64_t pipe_chunk, uint32_t slots,
                                         uint64_t direct_chunk, uint64_t push_chunk, uint64_t staged, uint64_t pull,
                                         nimbleItem* items, int cap, int* nitems) {
    return nb::guarded([&] {
        if (!nitems) throw std::invalid_argument("schedule: bad argument");
        nb::Schedule sc = nb::debug_schedule(p, rank, ranks, pipe_chunk, slots, direct_chunk, push_chunk, staged, pull);
        if (sc.cuts.size() + sc.ll_cuts.size() > static_cast<size_t>(nb::kMaxGenCuts))
            throw nb::Error(nimbleInvalidUsage, "schedule: more flows than the device generator takes");
        *nitems = static_cast<int>(sc.nitems);
        if (!items) return;
        auto check = [](cudaError_t e) {
            if (e != cudaSuccess) throw nb::Error(nimbleUnhandledCudaError, cudaGetErrorString(e));
        };
        nb::GenArgs g;
        std::memset(&g, 0, sizeof g);
        g.ncuts = g.nkeyed = static_cast<uint32_t>(sc.cuts.size());
        g.nitems = sc.nitems;
        std::copy(sc.cuts.begin(), sc.cuts.end(), g.cuts);
        nb::Item* d = nullptr;
        check(cudaMalloc(&d, std::max<size_t>(sc.nitems, 1) * sizeof(nb::Item)));
        check(cudaMemset(d, 0xff, std::max<size_t>(sc.nitems, 1) * sizeof(nb::Item)));
        g.items = d;
        cudaError_t e = nb::launch_gen(g, nullptr);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e == cudaSuccess)
            e = cudaMemcpy(items, d, std::min<size_t>(sc.nitems, cap > 0 ? cap : 0) * sizeof(nb::Item),
                           cudaMemcpyDeviceToHost);
        cudaFree(d);
        check(e);
    });
}

}  // extern "C"
