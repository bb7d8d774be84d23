// MCF-inspired multi-path planner (the paper's Algorithm 1).
//
// Reference semantics, kept bit-exact: proj/src/planner.cpp
//   routes_for      <- enumerate_paths   :39-108
//   CostParams      <- CostModel         planner.hpp:36-49, hop_penalty :12-19
//   mcf_plan        <- plan              :320-429 (sweep, refine_plan :131-300,
//                                                  direct-layout guard :395-419)
//   direct_plan     <- plan_direct_baseline :431-438
//   link_loads      <- plan_link_loads   :440-447
//   peak_load       <- max_normalized_load :449-455
//   plan_json       <- plan_to_json      :466-492
// All load and flow values are integer byte counts < 2^53 held in doubles, so
// the arithmetic is exact; the TU is compiled with -ffp-contract=off so the
// cost comparisons (max drain time + hop penalty) round exactly as there.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "demand.hpp"
#include "fabric.hpp"

namespace nb {

enum class Route : int { Direct = 0, TwoHop = 1, Rail = 2 };

constexpr int kMaxRouteEdges = 8;

struct Candidate {
    Route route = Route::Direct;
    int via = -1;    // relay GPU ordinal (TwoHop)
    int rail = -1;   // NIC index (Rail)
    int hops = 1;    // logical hop count seen by the penalty
    bool pair_direct = false;
    int ne = 0;
    int e[kMaxRouteEdges] = {};
};

struct CostParams {
    bool normalize = true;
    double pi = 0.25;
    std::uint64_t cutoff = 1ull << 20;      // detours forbidden at or below
    std::uint64_t sat_intra = 64ull << 20;  // penalty fades to zero here
    std::uint64_t sat_inter = 32ull << 20;
    double penalty(const Candidate& c, std::uint64_t message) const;
    static CostParams unpenalized();
};

struct PlanParams {
    double lambda = 0.5;
    std::uint64_t epsilon = 4ull << 20;
    CostParams cost;
    std::uint64_t max_visits = 1000000;
};

struct PlanCounters {
    std::uint64_t pair_visits = 0, placements = 0, fallback_pairs = 0, residual_flows = 0,
                  refine_moves = 0;
    double wall_seconds = 0.0;
};

struct Flow {
    int cand;
    double bytes;
};

struct PairRoutes {
    int src = -1, dst = -1;
    std::uint64_t demand = 0;
    std::vector<Candidate> cands;
    std::vector<Flow> flows;  // ascending candidate order
};

struct PlanResult {
    std::vector<PairRoutes> pairs;  // s-major, d-minor, zero demands skipped
    std::uint64_t epsilon = 4ull << 20;
    PlanCounters stats;
};

std::vector<Candidate> routes_for(const LinkModel& lm, int ranks, int rpn, int s, int d);
PlanResult mcf_plan(const LinkModel& lm, int ranks, int rpn, const Demand& m, const PlanParams& p);
PlanResult direct_plan(const LinkModel& lm, int ranks, int rpn, const Demand& m);
std::vector<double> link_loads(const LinkModel& lm, const PlanResult& p);
double peak_load(const LinkModel& lm, const PlanResult& p);
std::string plan_json(const PlanResult& p);
// plan_from_json (planner.cpp:494-539): routes re-enumerated on `lm`, flows
// matched by (class, via, rail), per-pair conservation checked within 0.5 B.
PlanResult plan_from_json(const LinkModel& lm, int ranks, int rpn, const std::string& text);

}  // namespace nb
