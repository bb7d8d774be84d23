// plan.json reader: the inverse of plan_json() (planner.cpp:494-539 semantics).
// A minimal JSON value parser (objects, arrays, numbers, strings, literals) is
// enough for the plan document; keys may come in any order.
#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "planner.hpp"

namespace nb {

namespace {

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    double num = 0;
    bool flag = false;
    std::string str;
    std::vector<Value> items;
    std::map<std::string, Value> fields;

    const Value& at(const std::string& k) const {
        auto it = fields.find(k);
        if (kind != Object || it == fields.end()) throw std::runtime_error("plan json: missing key '" + k + "'");
        return it->second;
    }
    bool has(const std::string& k) const { return kind == Object && fields.count(k); }
    double number() const {
        if (kind != Number) throw std::runtime_error("plan json: expected a number");
        return num;
    }
    std::uint64_t u64() const {
        const double v = number();
        if (v < 0 || v != std::floor(v)) throw std::runtime_error("plan json: expected a non-negative integer");
        return static_cast<std::uint64_t>(v);
    }
};

class Parser {
  public:
    explicit Parser(const std::string& t) : t_(t) {}
    Value document() {
        Value v = value();
        ws();
        if (p_ != t_.size()) fail("trailing characters");
        return v;
    }

  private:
    const std::string& t_;
    size_t p_ = 0;

    [[noreturn]] void fail(const char* what) {
        throw std::runtime_error(std::string("plan json parse error at ") + std::to_string(p_) + ": " + what);
    }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\r' || t_[p_] == '\t')) ++p_;
    }
    bool eat(char c) {
        ws();
        if (p_ < t_.size() && t_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    Value value() {
        ws();
        if (p_ >= t_.size()) fail("unexpected end");
        const char c = t_[p_];
        Value v;
        if (c == '{') {
            ++p_;
            v.kind = Value::Object;
            if (eat('}')) return v;
            do {
                ws();
                if (p_ >= t_.size() || t_[p_] != '"') fail("expected a key");
                std::string k = string();
                if (!eat(':')) fail("expected ':'");
                v.fields[k] = value();
            } while (eat(','));
            if (!eat('}')) fail("expected '}'");
        } else if (c == '[') {
            ++p_;
            v.kind = Value::Array;
            if (eat(']')) return v;
            do v.items.push_back(value());
            while (eat(','));
            if (!eat(']')) fail("expected ']'");
        } else if (c == '"') {
            v.kind = Value::String;
            v.str = string();
        } else if (t_.compare(p_, 4, "true") == 0 || t_.compare(p_, 5, "false") == 0) {
            v.kind = Value::Bool;
            v.flag = t_[p_] == 't';
            p_ += v.flag ? 4 : 5;
        } else if (t_.compare(p_, 4, "null") == 0) {
            p_ += 4;
        } else {
            char* end = nullptr;
            v.kind = Value::Number;
            v.num = std::strtod(t_.c_str() + p_, &end);
            if (end == t_.c_str() + p_) fail("bad value");
            p_ = static_cast<size_t>(end - t_.c_str());
        }
        return v;
    }
    std::string string() {
        std::string s;
        ++p_;  // opening quote
        while (p_ < t_.size() && t_[p_] != '"') {
            if (t_[p_] == '\\') {
                if (++p_ >= t_.size()) fail("bad escape");
            }
            s += t_[p_++];
        }
        if (p_ >= t_.size()) fail("unterminated string");
        ++p_;
        return s;
    }
};

Route route_of(const std::string& cls) {
    if (cls == "direct") return Route::Direct;
    if (cls == "intra_two_hop") return Route::TwoHop;
    if (cls == "inter_rail") return Route::Rail;
    throw std::runtime_error("plan: unknown route class '" + cls + "'");
}

}  // namespace

PlanResult plan_from_json(const LinkModel& lm, int ranks, int rpn, const std::string& text) {
    const Value doc = Parser(text).document();
    PlanResult p;
    p.epsilon = doc.has("epsilon") ? doc.at("epsilon").u64() : (4ull << 20);
    if (doc.has("stats")) {
        const Value& s = doc.at("stats");
        auto get = [&s](const char* k) { return s.has(k) ? s.at(k).u64() : 0ull; };
        p.stats.pair_visits = get("pair_visits");
        p.stats.placements = get("placements");
        p.stats.fallback_pairs = get("fallback_pairs");
        p.stats.residual_flows = get("residual_flows");
        p.stats.refine_moves = get("refine_moves");
        p.stats.wall_seconds = s.has("wall_seconds") ? s.at("wall_seconds").number() : 0.0;
    }
    for (const Value& pj : doc.at("pairs").items) {
        PairRoutes pr;
        pr.src = static_cast<int>(pj.at("src").number());
        pr.dst = static_cast<int>(pj.at("dst").number());
        pr.demand = pj.at("demand").u64();
        pr.cands = routes_for(lm, ranks, rpn, pr.src, pr.dst);
        double placed = 0.0;
        for (const Value& fj : pj.at("flows").items) {
            const Route r = route_of(fj.at("class").str);
            const int via = static_cast<int>(fj.at("via").number());
            const int rail = static_cast<int>(fj.at("rail").number());
            int found = -1;
            for (size_t c = 0; c < pr.cands.size() && found < 0; ++c)
                if (pr.cands[c].route == r && pr.cands[c].via == via && pr.cands[c].rail == rail)
                    found = static_cast<int>(c);
            if (found < 0)
                throw std::runtime_error("plan: flow references a route the topology lacks (pair " +
                                         std::to_string(pr.src) + "->" + std::to_string(pr.dst) + ", class " +
                                         fj.at("class").str + ")");
            const double bytes = fj.at("bytes").number();
            pr.flows.push_back({found, bytes});
            placed += bytes;
        }
        if (std::abs(placed - static_cast<double>(pr.demand)) > 0.5)
            throw std::runtime_error("plan: flows for pair " + std::to_string(pr.src) + "->" +
                                     std::to_string(pr.dst) + " do not sum to the demand");
        p.pairs.push_back(std::move(pr));
    }
    return p;
}

}  // namespace nb
