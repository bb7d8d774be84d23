// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A JSON-in / JSON-out C entry point over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp), compiled in place by oracle/Makefile into
// oracle/_ref/libnimble_ref.so.  tests/, __graft_entry__.smoke() and the
// bench.py reference arm are the only callers (through oracle/ref.py).
//
// Every operation is a straight call into the reference's public API:
//   gen       -> gen_p2p / gen_skewed_a2av / gen_irregular / gen_stencil_1d /
//                gen_aggregator                  (proj/src/workloads.cpp:46-152)
//   enumerate -> enumerate_paths                 (proj/src/planner.cpp:39-108)
//   plan      -> plan + plan_link_loads + max_normalized_load
//                                                (proj/src/planner.cpp:320-455)
//   direct    -> plan_direct_baseline            (proj/src/planner.cpp:431-438)
//   simulate  -> simulate_exchange               (proj/src/simulator.cpp:226-262)
//   transfer  -> simulate_transfer (+ trace)     (proj/src/pipeline.cpp:66-116)
//   topology  -> build_canonical link inventory  (proj/src/topology.cpp:119-179)
//   exact     -> solve_exact                     (proj/src/oracle.cpp:67-91)
//   calibrate -> calibrate with given targets    (proj/src/calibration.cpp:54-100)
//   multipath -> intra_multipath_speedup         (proj/src/calibration.cpp:11-23)
#include "nimble/calibration.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <json.hpp>

#include "nimble/oracle.hpp"
#include "nimble/pipeline.hpp"
#include "nimble/planner.hpp"
#include "nimble/simulator.hpp"
#include "nimble/topology.hpp"
#include "nimble/units.hpp"
#include "nimble/workloads.hpp"

using nlohmann::json;
using namespace nimble;

namespace {

Topology topo_from(const json& t) {
    std::string fab = t.value("fabric", std::string("nvswitch"));
    Fabric f = fab == "alltoall" ? Fabric::AllToAllNvLink : Fabric::NvSwitch;
    Topology topo = build_canonical(t.value("nodes", 1), t.value("gpus", 8), t.value("nics", 0),
                                    gbps(t.value("nvlink_gbps", 900.0)),
                                    gbps(t.value("rail_gbps", 50.0)), f);
    if (t.contains("capacity_overrides"))
        for (const auto& o : t.at("capacity_overrides"))
            topo.links[o.at(0).get<size_t>()].capacity = o.at(1).get<double>();
    return topo;
}

DemandMatrix demand_from(const json& w, int ranks) {
    std::string kind = w.at("kind").get<std::string>();
    if (kind == "p2p")
        return gen_p2p(ranks, w.value("src", 0), w.value("dst", 1), w.at("size").get<std::uint64_t>());
    if (kind == "skewed")
        return gen_skewed_a2av(ranks, w.at("size").get<std::uint64_t>(), w.at("ratio").get<double>(),
                               w.value("hot", 0), w.value("seed", std::uint64_t{0}),
                               w.value("per_sender_hot", false));
    if (kind == "irregular")
        return gen_irregular(ranks, w.at("size").get<std::uint64_t>(), w.at("sparsity").get<double>(),
                             w.at("seed").get<std::uint64_t>());
    if (kind == "stencil") return gen_stencil_1d(ranks, w.at("size").get<std::uint64_t>());
    if (kind == "aggregator")
        return gen_aggregator(ranks, w.at("dsts").get<std::vector<int>>(),
                              w.at("size").get<std::uint64_t>());
    if (kind == "matrix") {
        DemandMatrix m;
        m.ranks = ranks;
        m.bytes = w.at("bytes").get<std::vector<std::uint64_t>>();
        m.validate();
        return m;
    }
    throw std::runtime_error("unknown workload kind " + kind);
}

PlannerConfig planner_from(const json& req) {
    PlannerConfig pc;
    if (!req.contains("planner")) return pc;
    const json& p = req.at("planner");
    pc.lambda = p.value("lambda", pc.lambda);
    pc.epsilon = p.value("epsilon", pc.epsilon);
    pc.cost.pi = p.value("pi", pc.cost.pi);
    pc.cost.small_message_cutoff = p.value("small_message_cutoff", pc.cost.small_message_cutoff);
    pc.cost.saturation_intra = p.value("saturation_intra", pc.cost.saturation_intra);
    pc.cost.saturation_inter = p.value("saturation_inter", pc.cost.saturation_inter);
    pc.max_pair_visits = p.value("max_pair_visits", pc.max_pair_visits);
    if (p.value("unpenalized", false)) pc.cost = CostModel::unpenalized();
    return pc;
}

PipelineConfig pipeline_from(const json& req) {
    PipelineConfig cfg;
    if (!req.contains("pipeline")) return cfg;
    const json& p = req.at("pipeline");
    if (p.value("ideal", false)) return PipelineConfig::ideal();
    cfg.p2p_buffer = p.value("p2p_buffer", cfg.p2p_buffer);
    cfg.pipe_chunk = p.value("pipe_chunk", cfg.pipe_chunk);
    cfg.hop_latency = p.value("hop_latency", cfg.hop_latency);
    cfg.nic_hop_latency = p.value("nic_hop_latency", cfg.nic_hop_latency);
    cfg.channels_per_peer = p.value("channels_per_peer", cfg.channels_per_peer);
    return cfg;
}

const char* cls_name(PathClass c) {
    switch (c) {
    case PathClass::Direct: return "direct";
    case PathClass::IntraTwoHop: return "intra_two_hop";
    case PathClass::InterRail: return "inter_rail";
    }
    return "?";
}

json plan_doc(const Topology& topo, const Plan& p) {
    json j;
    j["plan"] = plan_to_json(p);
    // candidate index of each flow, so parity does not rely on class/via only
    json cand = json::array();
    for (const PairPlan& pp : p.pairs) {
        json fl = json::array();
        for (const FlowAssignment& f : pp.flows) fl.push_back(f.candidate);
        cand.push_back(fl);
    }
    j["flow_candidates"] = cand;
    j["loads"] = plan_link_loads(topo, p);
    j["max_norm_load"] = max_normalized_load(topo, p);
    return j;
}

json run(const json& req) {
    std::string op = req.at("op").get<std::string>();
    json out;
    if (op == "calibrate") {  // calibrate() with caller-supplied targets (proj/src/calibration.cpp:54-100)
        CalibrationTargets t;
        const json& q = req.at("targets");
        t.one_intermediate = q.value("one_intermediate", t.one_intermediate);
        t.two_intermediate = q.value("two_intermediate", t.two_intermediate);
        t.four_rail = q.value("four_rail", t.four_rail);
        t.message = q.value("message", t.message);
        t.nvlink_gbps = q.value("nvlink_gbps", t.nvlink_gbps);
        t.rail_gbps = q.value("rail_gbps", t.rail_gbps);
        CalibrationResult r = calibrate(t);
        out["hop_latency"] = r.config.hop_latency;
        out["pi"] = r.pi;
        out["one_intermediate"] = r.one_intermediate;
        out["two_intermediate"] = r.two_intermediate;
        out["four_rail"] = r.four_rail;
        return out;
    }
    if (op == "multipath") {  // intra_multipath_speedup (proj/src/calibration.cpp:11-23)
        PipelineConfig cfg;
        cfg.hop_latency = req.value("hop_latency", cfg.hop_latency);
        out["speedup"] = intra_multipath_speedup(req.at("intermediates").get<int>(), req.at("message").get<std::uint64_t>(),
                                                 req.at("nvlink_gbps").get<double>(), cfg);
        return out;
    }
    if (op == "topology") {
        Topology t = topo_from(req.at("topology"));
        json links = json::array();
        for (const Link& l : t.links)
            links.push_back({{"id", l.id}, {"name", t.link_name(l.id)}, {"capacity", l.capacity},
                             {"kind", static_cast<int>(l.kind)}});
        out["links"] = links;
        out["text"] = save_topology(t);
        return out;
    }
    if (op == "transfer") {
        std::vector<HopSpec> chain;
        for (const auto& h : req.at("chain")) chain.push_back({h.at(0).get<double>(), h.at(1).get<double>()});
        TransferTrace tr;
        double c = simulate_transfer(chain, req.at("bytes").get<double>(), pipeline_from(req), &tr);
        out["completion"] = c;
        out["chunk_bytes"] = tr.chunk_bytes;
        out["start"] = tr.start;
        out["tx_done"] = tr.tx_done;
        out["delivered"] = tr.delivered;
        return out;
    }
    int ranks = req.at("ranks").get<int>();
    DemandMatrix d = demand_from(req.at("workload"), ranks);
    out["matrix"] = d.bytes;
    if (op == "gen") return out;
    Topology topo = topo_from(req.at("topology"));
    RankMap map = make_rank_map(ranks, req.value("ranks_per_node", topo.gpus_per_node));
    if (op == "enumerate") {
        json pairs = json::array();
        for (int s = 0; s < ranks; ++s)
            for (int t = 0; t < ranks; ++t) {
                if (s == t) continue;
                json cands = json::array();
                for (const CandidatePath& c : enumerate_paths(topo, map, s, t))
                    cands.push_back({{"class", cls_name(c.cls)}, {"via", c.via}, {"rail", c.rail},
                                     {"hops", c.hops}, {"pair_direct", c.pair_direct},
                                     {"edges", c.edges}});
                pairs.push_back({{"src", s}, {"dst", t}, {"candidates", cands}});
            }
        out["pairs"] = pairs;
        return out;
    }
    if (op == "plan" || op == "direct" || op == "simulate") {
        Plan p = op == "direct" ? plan_direct_baseline(topo, map, d)
                                : plan(topo, map, d, planner_from(req));
        p.stats.wall_seconds = 0.0;
        json doc = plan_doc(topo, p);
        for (auto it = doc.begin(); it != doc.end(); ++it) out[it.key()] = it.value();
        Plan base = plan_direct_baseline(topo, map, d);
        out["direct_max_norm_load"] = max_normalized_load(topo, base);
        if (op == "simulate") {
            SimMode mode = parse_sim_mode(req.value("mode", std::string("closed_form")));
            PipelineConfig cfg = pipeline_from(req);
            ExchangeResult rn = simulate_exchange(topo, p, cfg, mode);
            ExchangeResult rb = simulate_exchange(topo, base, cfg, mode);
            out["completion"] = rn.completion;
            out["baseline_completion"] = rb.completion;
            out["speedup"] = speedup(rn, rb);
            out["link_bytes"] = rn.link_bytes;
            out["bottleneck_link"] = rn.bottleneck_link;
            double total = static_cast<double>(d.total());
            out["model_gbps"] = rn.completion > 0 ? total / rn.completion / 1e9 : 0.0;
        }
        return out;
    }
    if (op == "exact") {
        ExactInstance inst;
        inst.epsilon = req.value("epsilon", inst.epsilon);
        for (int s = 0; s < ranks; ++s)
            for (int t = 0; t < ranks; ++t)
                if (d.at(s, t)) inst.demands.push_back({s, t, static_cast<int>(d.at(s, t) / inst.epsilon)});
        ExactResult r = solve_exact(topo, map, inst);
        out["z_star"] = r.z_star;
        return out;
    }
    throw std::runtime_error("unknown op " + op);
}

} // namespace

extern "C" {

// Returns 0 and the response document, or 1 and {"error": "..."}.  When the
// document does not fit in `cap` bytes, *need holds the size to retry with.
int nref_call(const char* request, char* out, size_t cap, size_t* need) {
    std::string s;
    int rc = 0;
    try {
        s = run(json::parse(request)).dump();
    } catch (const std::exception& e) {
        s = json{{"error", e.what()}}.dump();
        rc = 1;
    }
    *need = s.size() + 1;
    if (s.size() + 1 > cap) return 2;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return rc;
}

// Wall time of plan() on the request's workload, `warmup` untimed calls then
// the median of `runs` timed ones (the cmd_bench protocol, tools/nimble.cpp:385-403).
double nref_time_plan(const char* request, int warmup, int runs) {
    try {
        json req = json::parse(request);
        int ranks = req.at("ranks").get<int>();
        DemandMatrix d = demand_from(req.at("workload"), ranks);
        Topology topo = topo_from(req.at("topology"));
        RankMap map = make_rank_map(ranks, req.value("ranks_per_node", topo.gpus_per_node));
        PlannerConfig pc = planner_from(req);
        for (int i = 0; i < warmup; ++i) plan(topo, map, d, pc);
        std::vector<double> t;
        for (int i = 0; i < runs; ++i) t.push_back(plan(topo, map, d, pc).stats.wall_seconds);
        std::sort(t.begin(), t.end());
        return t.empty() ? 0.0 : t[t.size() / 2];
    } catch (...) {
        return -1.0;
    }
}

// Plan once and export the flows as flat arrays for the CPU data-movement
// baseline: per flow (src, dst, via, bytes); returns the flow count or -1.
int nref_plan_flows(const char* request, int* src, int* dst, int* via, double* bytes, int cap) {
    try {
        json req = json::parse(request);
        int ranks = req.at("ranks").get<int>();
        DemandMatrix d = demand_from(req.at("workload"), ranks);
        Topology topo = topo_from(req.at("topology"));
        RankMap map = make_rank_map(ranks, req.value("ranks_per_node", topo.gpus_per_node));
        Plan p = plan(topo, map, d, planner_from(req));
        int n = 0;
        for (const PairPlan& pp : p.pairs)
            for (const FlowAssignment& f : pp.flows) {
                if (n >= cap) return -1;
                src[n] = pp.src;
                dst[n] = pp.dst;
                via[n] = pp.candidates[static_cast<size_t>(f.candidate)].via;
                bytes[n] = f.bytes;
                ++n;
            }
        return n;
    } catch (...) {
        return -1;
    }
}

} // extern "C"
