// MCF-inspired multi-path planner; see planner.hpp for the reference mapping.
#include "planner.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace nb {

double CostParams::penalty(const Candidate& c, std::uint64_t message) const {
    if (c.hops <= 1) return 0.0;
    if (message <= cutoff) return std::numeric_limits<double>::infinity();
    const std::uint64_t sat = c.route == Route::Rail ? sat_inter : sat_intra;
    const double fade = 1.0 - static_cast<double>(message) / static_cast<double>(sat);
    if (fade <= 0.0) return 0.0;
    return pi * static_cast<double>(c.hops - 1) * fade;
}

CostParams CostParams::unpenalized() {
    CostParams c;
    c.pi = 0.0;
    c.cutoff = 0;
    return c;
}

namespace {

void put(Candidate& c, int edge) {
    if (c.ne == kMaxRouteEdges) throw std::logic_error("route longer than kMaxRouteEdges");
    c.e[c.ne++] = edge;
}

// GPU a -> GPU b inside `node`: one mesh link, or up-port + down-port.
void intra(const LinkModel& lm, int node, int a, int b, Candidate& c) {
    if (a == b) return;
    if (lm.fabric == FabricKind::AllToAll) {
        put(c, lm.mesh(node, a, b));
    } else {
        put(c, lm.up(node, a));
        put(c, lm.down(node, b));
    }
}

// Per-link loads with their normalized drain times kept alongside, so the
// refinement's repeated "global max" is a plain max over cached quotients
// (identical values to recomputing load/capacity each time).
struct LoadBook {
    const LinkModel& lm;
    std::vector<double> load, drain;
    // Links whose drain is >= bar, kept current by add(): "peak() < bar" is
    // then "nhot == 0" in O(1) -- the refiner's trial moves touch <= 4 links.
    double bar = std::numeric_limits<double>::infinity();
    int nhot = 0;
    explicit LoadBook(const LinkModel& m) : lm(m), load(m.cap.size(), 0.0), drain(m.cap.size(), 0.0) {}
    void add(int e, double x) {
        const bool was = drain[e] >= bar;
        load[e] += x;
        drain[e] = load[e] / lm.cap[e];
        nhot += static_cast<int>(drain[e] >= bar) - static_cast<int>(was);
    }
    void set_bar(double b) {
        bar = b;
        nhot = 0;
        for (double v : drain) nhot += v >= b;
    }
    void add_route(const Candidate& c, double x) {
        for (int k = 0; k < c.ne; ++k) add(c.e[k], x);
    }
    double peak() const {
        double w = 0.0;
        for (double v : drain) w = std::max(w, v);
        return w;
    }
    bool touches_peak(const Candidate& c, double bar) const {
        for (int k = 0; k < c.ne; ++k)
            if (drain[c.e[k]] >= bar) return true;
        return false;
    }
    void reset(const std::vector<double>& l) {
        load = l;
        for (size_t e = 0; e < load.size(); ++e) drain[e] = load[e] / lm.cap[e];
        set_bar(bar);
    }
};

// max over the route's links of the (normalized) load after adding `pending`
double route_load_cost(const Candidate& c, const LoadBook& book, const CostParams& cost, double pending) {
    double worst = 0.0;
    for (int k = 0; k < c.ne; ++k) {
        const int e = c.e[k];
        const double v = cost.normalize ? (book.load[e] + pending) / book.lm.cap[e] : book.load[e] + pending;
        worst = std::max(worst, v);
    }
    return worst;
}

double route_cost(const Candidate& c, const LoadBook& book, const CostParams& cost,
                  std::uint64_t message, double pending) {
    return route_load_cost(c, book, cost, pending) + cost.penalty(c, message);
}

constexpr size_t kMaxCands = 64;  // routes per pair whose penalties the sweep caches

std::vector<PairRoutes> active_pairs(const LinkModel& lm, int ranks, int rpn, const Demand& m) {
    m.check();
    if (m.ranks != ranks) throw std::runtime_error("planner: matrix size does not match rank count");
    std::vector<PairRoutes> out;
    for (int s = 0; s < ranks; ++s)
        for (int d = 0; d < ranks; ++d) {
            const std::uint64_t b = m.at(s, d);
            if (!b) continue;
            PairRoutes pr;
            pr.src = s;
            pr.dst = d;
            pr.demand = b;
            pr.cands = routes_for(lm, ranks, rpn, s, d);
            out.push_back(std::move(pr));
        }
    return out;
}

// Chunk-move clean-up after the sweep (planner.cpp:122-300): reduce shifts a
// chunk off a bottleneck link when a sibling route strictly lowers the peak,
// consolidate walks detour chunks back to the direct route while that stays
// under the peak, eject resolves two-pair traps.  Penalties never rise.
class Refiner {
  public:
    Refiner(const LinkModel& lm, const std::vector<PairRoutes>& pairs,
            std::vector<std::vector<double>>& acc, LoadBook& book, const PlanParams& p)
        : pairs_(pairs), acc_(acc), book_(book), p_(p), eps_(static_cast<double>(p.epsilon)) {
        (void)lm;
        pens_.resize(pairs.size());
        for (size_t i = 0; i < pairs.size(); ++i)
            for (const Candidate& c : pairs[i].cands) pens_[i].push_back(p.cost.penalty(c, pairs[i].demand));
    }

    std::uint64_t run() {
        bool choice = false;  // with one route per pair no move exists (e.g. the nvswitch model)
        for (const PairRoutes& pr : pairs_) choice |= pr.cands.size() > 1;
        if (!choice) return 0;
        for (int round = 0; round < 8; ++round) {
            const bool r = reduce();
            const bool c = consolidate();
            if (!r && !c && !eject()) break;
        }
        return moves_;
    }

  private:
    static constexpr std::uint64_t kMoveCap = 4096;
    static constexpr int kEjectCap = 4096;

    const std::vector<PairRoutes>& pairs_;
    std::vector<std::vector<double>>& acc_;
    LoadBook& book_;
    const PlanParams& p_;
    const double eps_;
    std::vector<std::vector<double>> pens_;  // hop penalty per (pair, route): constant during refinement
    std::uint64_t moves_ = 0;
    int ejects_ = 0;

    void move(size_t i, size_t from, size_t to, double q) {
        book_.add_route(pairs_[i].cands[from], -q);
        book_.add_route(pairs_[i].cands[to], q);
        acc_[i][from] -= q;
        acc_[i][to] += q;
    }
    double pen(size_t i, size_t c) const { return pens_[i][c]; }

    bool reduce() {
        bool any = false;
        for (bool progress = true; progress && moves_ < kMoveCap;) {
            progress = false;
            const double cur = book_.peak();
            if (cur <= 0.0) break;
            const double bar = cur * (1.0 - 1e-12);
            book_.set_bar(bar);
            for (size_t i = 0; i < pairs_.size() && !progress; ++i) {
                const auto& cs = pairs_[i].cands;
                for (size_t c = 0; c < cs.size() && !progress; ++c) {
                    if (acc_[i][c] <= 0.0 || !book_.touches_peak(cs[c], bar)) continue;
                    const double q = std::min(eps_, acc_[i][c]);
                    const double pc = pen(i, c);
                    for (size_t a = 0; a < cs.size(); ++a) {
                        if (a == c || pen(i, a) > pc) continue;
                        move(i, c, a, q);
                        if (book_.nhot == 0) {  // peak() < bar
                            ++moves_;
                            progress = any = true;
                            break;
                        }
                        move(i, a, c, q);
                    }
                }
            }
        }
        return any;
    }

    bool consolidate() {
        bool any = false;
        for (bool progress = true; progress && moves_ < kMoveCap;) {
            progress = false;
            double cur = book_.peak();
            double bar = cur * (1.0 - 1e-12);
            for (size_t i = 0; i < pairs_.size(); ++i) {
                const auto& cs = pairs_[i].cands;
                for (size_t c = 1; c < cs.size(); ++c) {
                    while (acc_[i][c] > 0.0 && moves_ < kMoveCap) {
                        const double q = std::min(eps_, acc_[i][c]);
                        move(i, c, 0, q);
                        if (book_.touches_peak(cs[0], bar)) {
                            move(i, 0, c, q);
                            break;
                        }
                        ++moves_;
                        progress = any = true;
                        const double now = book_.peak();
                        if (now < cur) {
                            cur = now;
                            bar = cur * (1.0 - 1e-12);
                        }
                    }
                }
            }
        }
        return any;
    }

    bool eject() {
        if (moves_ + 2 > kMoveCap) return false;
        const double cur = book_.peak();
        if (cur <= 0.0) return false;
        const double bar = cur * (1.0 - 1e-12);
        book_.set_bar(bar);
        for (size_t i = 0; i < pairs_.size(); ++i) {
            const auto& cs = pairs_[i].cands;
            for (size_t c = 0; c < cs.size(); ++c) {
                if (acc_[i][c] <= 0.0 || !book_.touches_peak(cs[c], bar)) continue;
                const double q = std::min(eps_, acc_[i][c]);
                const double pc = pen(i, c);
                for (size_t a = 0; a < cs.size(); ++a) {
                    if (a == c || pen(i, a) > pc) continue;
                    move(i, c, a, q);
                    for (int k = 0; k < cs[a].ne; ++k) {
                        const int hot = cs[a].e[k];
                        if (book_.drain[hot] < bar) continue;
                        if (evict_from(hot, i, a, c)) return true;
                    }
                    move(i, a, c, q);
                    if (ejects_ >= kEjectCap) return false;
                }
            }
        }
        return false;
    }

    // Try to move one chunk of some other route that crosses link `hot` to a
    // sibling route of its own pair, so the peak drops below `bar`.
    bool evict_from(int hot, size_t i, size_t a, size_t c) {  // the book's bar is eject()'s
        for (size_t j = 0; j < pairs_.size(); ++j) {
            const auto& js = pairs_[j].cands;
            for (size_t d = 0; d < js.size(); ++d) {
                if (j == i && (d == a || d == c)) continue;
                if (acc_[j][d] <= 0.0) continue;
                if (std::find(js[d].e, js[d].e + js[d].ne, hot) == js[d].e + js[d].ne) continue;
                const double v = std::min(eps_, acc_[j][d]);
                const double pd = pen(j, d);
                for (size_t b = 0; b < js.size(); ++b) {
                    if (b == d || pen(j, b) > pd) continue;
                    if (ejects_ >= kEjectCap) break;
                    ++ejects_;
                    move(j, d, b, v);
                    if (book_.nhot == 0) {  // peak() < bar (set_bar in eject)
                        moves_ += 2;
                        return true;
                    }
                    move(j, b, d, v);
                }
            }
        }
        return false;
    }
};

}  // namespace

std::vector<Candidate> routes_for(const LinkModel& lm, int ranks, int rpn, int s, int d) {
    if (s < 0 || s >= ranks || d < 0 || d >= ranks) throw std::runtime_error("enumerate_paths: rank out of range");
    if (s == d) throw std::runtime_error("enumerate_paths: src equals dst");
    if (rpn < 1) throw std::runtime_error("rank map: ranks and ranks_per_node must be >= 1");
    const int sn = s / rpn, so = s % rpn, dn = d / rpn, dg = d % rpn;
    if (sn >= lm.nodes || dn >= lm.nodes || so >= lm.gpus || dg >= lm.gpus)
        throw std::runtime_error("enumerate_paths: rank map exceeds topology");
    std::vector<Candidate> out;
    if (sn == dn) {
        Candidate direct;
        direct.pair_direct = true;
        intra(lm, sn, so, dg, direct);
        out.push_back(direct);
        if (lm.fabric == FabricKind::AllToAll)
            for (int v = 0; v < lm.gpus; ++v) {
                if (v == so || v == dg) continue;
                Candidate relay;
                relay.route = Route::TwoHop;
                relay.via = v;
                relay.hops = 2;
                put(relay, lm.mesh(sn, so, v));
                put(relay, lm.mesh(sn, v, dg));
                out.push_back(relay);
            }
        return out;
    }
    if (lm.nics == 0) throw std::runtime_error("enumerate_paths: no rails between nodes");
    auto via_rail = [&](int r) {
        Candidate c;
        c.route = Route::Rail;
        c.rail = r;
        c.hops = 1 + (so != r) + (dg != r);
        intra(lm, sn, so, r, c);
        put(c, lm.attach_up(sn, r));
        put(c, lm.rail(sn, dn, r));
        put(c, lm.attach_down(dn, r));
        intra(lm, dn, r, dg, c);
        return c;
    };
    // the destination's own rail is the designated direct route (planner.cpp:95-102)
    const int home = dg % lm.nics;
    Candidate direct = via_rail(home);
    direct.pair_direct = true;
    direct.hops = 1;
    out.push_back(direct);
    for (int r = 0; r < lm.nics; ++r)
        if (r != home) out.push_back(via_rail(r));
    return out;
}

PlanResult mcf_plan(const LinkModel& lm, int ranks, int rpn, const Demand& m, const PlanParams& p) {
    if (!(p.lambda > 0.0 && p.lambda <= 1.0)) throw std::runtime_error("planner: lambda must be in (0,1]");
    if (p.epsilon == 0) throw std::runtime_error("planner: epsilon must be positive");
    const auto t0 = std::chrono::steady_clock::now();
    PlanResult res;
    res.epsilon = p.epsilon;
    res.pairs = active_pairs(lm, ranks, rpn, m);
    const size_t n = res.pairs.size();
    LoadBook book(lm);
    std::vector<std::vector<double>> acc(n);
    std::vector<double> left(n);
    std::vector<size_t> live(n);
    for (size_t i = 0; i < n; ++i) {
        acc[i].assign(res.pairs[i].cands.size(), 0.0);
        left[i] = static_cast<double>(res.pairs[i].demand);
        live[i] = i;
    }

    // Sweep: each visit routes lambda of the pair's remaining bytes (whole
    // epsilon chunks, at least one) chunk by chunk onto the cheapest route.
    const double eps = static_cast<double>(p.epsilon);
    bool exhausted = false;
    while (!live.empty() && !exhausted) {
        std::vector<size_t> next;
        for (size_t i : live) {
            if (res.stats.pair_visits >= p.max_visits) {
                exhausted = true;
                next.push_back(i);
                continue;
            }
            ++res.stats.pair_visits;
            const PairRoutes& pr = res.pairs[i];
            double r = left[i];
            double budget = r < eps ? r : std::max(eps, std::floor(r * p.lambda / eps) * eps);
            if (pr.cands.size() == 1 && budget > 0.0) {
                // One route: every chunk of the visit lands on it.  Loads are
                // integer-valued doubles below 2^53, so adding the visit at once
                // leaves the same loads, flows and counts as chunk by chunk.
                const double full = std::floor(budget / eps);
                const bool tail = budget - full * eps > 0.0;
                book.add_route(pr.cands[0], budget);
                acc[i][0] += budget;
                res.stats.placements += static_cast<std::uint64_t>(full) + (tail ? 1 : 0);
                if (tail) ++res.stats.residual_flows;
                r -= budget;
                budget = 0.0;
            }
            // the hop penalty depends on the route and the pair's demand only
            double pens[kMaxCands];
            const size_t nc = std::min(pr.cands.size(), kMaxCands);
            if (budget > 0.0)
                for (size_t c = 0; c < nc; ++c) pens[c] = p.cost.penalty(pr.cands[c], pr.demand);
            while (budget > 0.0) {
                const double chunk = std::min(eps, budget);
                size_t best = 0;
                double best_cost = std::numeric_limits<double>::infinity();
                for (size_t c = 0; c < pr.cands.size(); ++c) {
                    const double cost = c < nc ? route_load_cost(pr.cands[c], book, p.cost, chunk) + pens[c]
                                               : route_cost(pr.cands[c], book, p.cost, pr.demand, chunk);
                    if (cost < best_cost) {
                        best_cost = cost;
                        best = c;
                    }
                }
                book.add_route(pr.cands[best], chunk);
                acc[i][best] += chunk;
                ++res.stats.placements;
                if (chunk < eps) ++res.stats.residual_flows;
                budget -= chunk;
                r -= chunk;
            }
            left[i] = r;
            if (r > 0.0) next.push_back(i);
        }
        live.swap(next);
    }
    if (exhausted) {  // visit cap hit: the rest ships on the direct route
        for (size_t i : live) {
            acc[i][0] += left[i];
            book.add_route(res.pairs[i].cands[0], left[i]);
            ++res.stats.fallback_pairs;
        }
    }
    res.stats.refine_moves = Refiner(lm, res.pairs, acc, book, p).run();

    // Guard: never lose to the all-direct layout (planner.cpp:395-419).
    std::vector<double> direct(lm.cap.size(), 0.0);
    for (const PairRoutes& pr : res.pairs)
        for (int k = 0; k < pr.cands[0].ne; ++k) direct[pr.cands[0].e[k]] += static_cast<double>(pr.demand);
    LoadBook dbook(lm);
    dbook.reset(direct);
    if (book.peak() > dbook.peak() * (1.0 + 1e-12)) {
        for (size_t i = 0; i < n; ++i) {
            acc[i].assign(res.pairs[i].cands.size(), 0.0);
            acc[i][0] = static_cast<double>(res.pairs[i].demand);
        }
        book.reset(direct);
        res.stats.refine_moves += Refiner(lm, res.pairs, acc, book, p).run();
    }
    for (size_t i = 0; i < n; ++i)
        for (size_t c = 0; c < acc[i].size(); ++c)
            if (acc[i][c] > 0.0) res.pairs[i].flows.push_back({static_cast<int>(c), acc[i][c]});
    res.stats.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return res;
}

PlanResult direct_plan(const LinkModel& lm, int ranks, int rpn, const Demand& m) {
    PlanResult res;
    res.pairs = active_pairs(lm, ranks, rpn, m);
    for (PairRoutes& pr : res.pairs) pr.flows.push_back({0, static_cast<double>(pr.demand)});
    return res;
}

std::vector<double> link_loads(const LinkModel& lm, const PlanResult& p) {
    std::vector<double> l(lm.cap.size(), 0.0);
    for (const PairRoutes& pr : p.pairs)
        for (const Flow& f : pr.flows) {
            const Candidate& c = pr.cands[static_cast<size_t>(f.cand)];
            for (int k = 0; k < c.ne; ++k) l[c.e[k]] += f.bytes;
        }
    return l;
}

double peak_load(const LinkModel& lm, const PlanResult& p) {
    const std::vector<double> l = link_loads(lm, p);
    double w = 0.0;
    for (size_t e = 0; e < l.size(); ++e) w = std::max(w, l[e] / lm.cap[e]);
    return w;
}

namespace {

std::string num(double v) {
    std::string s = shortest_double(v);
    if (std::isfinite(v) && s.find_first_of(".eE") == std::string::npos) s += ".0";
    return s;
}

const char* route_name(Route r) {
    return r == Route::Direct ? "direct" : r == Route::TwoHop ? "intra_two_hop" : "inter_rail";
}

}  // namespace

std::string plan_json(const PlanResult& p) {
    std::string s = "{\"epsilon\":" + std::to_string(p.epsilon) + ",\"stats\":{";
    s += "\"pair_visits\":" + std::to_string(p.stats.pair_visits);
    s += ",\"placements\":" + std::to_string(p.stats.placements);
    s += ",\"fallback_pairs\":" + std::to_string(p.stats.fallback_pairs);
    s += ",\"residual_flows\":" + std::to_string(p.stats.residual_flows);
    s += ",\"refine_moves\":" + std::to_string(p.stats.refine_moves);
    s += ",\"wall_seconds\":" + num(p.stats.wall_seconds) + "},\"pairs\":[";
    for (size_t i = 0; i < p.pairs.size(); ++i) {
        const PairRoutes& pr = p.pairs[i];
        if (i) s += ',';
        s += "{\"src\":" + std::to_string(pr.src) + ",\"dst\":" + std::to_string(pr.dst) +
             ",\"demand\":" + std::to_string(pr.demand) + ",\"flows\":[";
        for (size_t f = 0; f < pr.flows.size(); ++f) {
            const Candidate& c = pr.cands[static_cast<size_t>(pr.flows[f].cand)];
            if (f) s += ',';
            s += std::string("{\"class\":\"") + route_name(c.route) + "\",\"via\":" + std::to_string(c.via) +
                 ",\"rail\":" + std::to_string(c.rail) + ",\"bytes\":" + num(pr.flows[f].bytes) + "}";
        }
        s += "]}";
    }
    return s + "]}";
}

}  // namespace nb
