// Link-load model construction and lookups; see fabric.hpp.
// Reference semantics: proj/src/topology.cpp (ids :83-117, construction
// :119-179, invariants :181-252, file format :296-403).
#include "fabric.hpp"

#include <charconv>
#include <cstdio>
#include <sstream>
#include <stdexcept>

namespace nb {

namespace {
constexpr int kGpu = 0, kNic = 1, kHub = 2;
}

int LinkModel::mesh(int node, int a, int b) const {
    if (fabric != FabricKind::AllToAll || a == b) throw std::logic_error("nvlink_id: no such link");
    return node * intra_per_node() + a * (gpus - 1) + (b < a ? b : b - 1);
}

int LinkModel::up(int node, int g) const {
    if (fabric != FabricKind::NvSwitch) throw std::logic_error("port_up_id: wrong fabric");
    return node * intra_per_node() + g;
}

int LinkModel::down(int node, int g) const {
    if (fabric != FabricKind::NvSwitch) throw std::logic_error("port_down_id: wrong fabric");
    return node * intra_per_node() + gpus + g;
}

int LinkModel::attach_up(int node, int nic) const {
    if (nic < 0 || nic >= nics) throw std::logic_error("attach_up_id: bad nic");
    return nodes * intra_per_node() + 2 * (node * nics + nic);
}

int LinkModel::rail(int a, int b, int r) const {
    if (a == b || r < 0 || r >= nics) throw std::logic_error("rail_id: no such rail");
    const int ordered_pair = a * (nodes - 1) + (b < a ? b : b - 1);
    return nodes * intra_per_node() + 2 * nodes * nics + ordered_pair * nics + r;
}

int LinkModel::find(const Endpoint& a, const Endpoint& b) const {
    for (int i = 0; i < links(); ++i)
        if (from[i] == a && to[i] == b) return i;
    return -1;
}

std::string endpoint_name(const Endpoint& e) {
    char buf[40];
    if (e.kind == kGpu) std::snprintf(buf, sizeof buf, "n%d.g%d", e.node, e.index);
    else if (e.kind == kNic) std::snprintf(buf, sizeof buf, "n%d.nic%d", e.node, e.index);
    else std::snprintf(buf, sizeof buf, "n%d.sw", e.node);
    return buf;
}

std::string LinkModel::name(int id) const {
    return endpoint_name(from[id]) + "->" + endpoint_name(to[id]);
}

LinkModel make_link_model(int nodes, int gpus, int nics, double nvlink_cap, double rail_cap,
                          FabricKind fabric) {
    if (nodes < 1) throw std::runtime_error("build_canonical: nodes must be >= 1");
    if (gpus < 1) throw std::runtime_error("build_canonical: gpus_per_node must be >= 1");
    if (nics < 0 || nics > gpus)
        throw std::runtime_error("build_canonical: nics_per_node must be in [0, gpus_per_node]");
    if (!(nvlink_cap > 0)) throw std::runtime_error("build_canonical: nvlink capacity must be positive");
    if (nics > 0 && !(rail_cap > 0))
        throw std::runtime_error("build_canonical: rail capacity must be positive when NICs are present");
    LinkModel m;
    m.nodes = nodes;
    m.gpus = gpus;
    m.nics = nics;
    m.fabric = fabric;
    m.nvlink_cap = nvlink_cap;
    m.rail_cap = rail_cap;
    auto push = [&m](Endpoint a, Endpoint b, LinkClass c, double bw) {
        m.from.push_back(a);
        m.to.push_back(b);
        m.cls.push_back(c);
        m.cap.push_back(bw);
    };
    for (int n = 0; n < nodes; ++n) {
        if (fabric == FabricKind::AllToAll) {
            for (int a = 0; a < gpus; ++a)
                for (int b = 0; b < gpus; ++b)
                    if (a != b) push({n, kGpu, a}, {n, kGpu, b}, LinkClass::NvLink, nvlink_cap);
        } else {
            for (int g = 0; g < gpus; ++g) push({n, kGpu, g}, {n, kHub, 0}, LinkClass::SwitchPort, nvlink_cap);
            for (int g = 0; g < gpus; ++g) push({n, kHub, 0}, {n, kGpu, g}, LinkClass::SwitchPort, nvlink_cap);
        }
    }
    for (int n = 0; n < nodes; ++n)
        for (int k = 0; k < nics; ++k) {
            push({n, kGpu, k}, {n, kNic, k}, LinkClass::Attach, 2 * rail_cap);
            push({n, kNic, k}, {n, kGpu, k}, LinkClass::Attach, 2 * rail_cap);
        }
    for (int a = 0; a < nodes; ++a)
        for (int b = 0; b < nodes; ++b)
            if (a != b)
                for (int r = 0; r < nics; ++r) push({a, kNic, r}, {b, kNic, r}, LinkClass::Rail, rail_cap);
    m.check();
    return m;
}

void LinkModel::check() const {
    auto fail = [](const std::string& why) { throw std::runtime_error("topology invariant: " + why); };
    if (nodes < 1 || gpus < 1) fail("empty topology");
    if (nics < 0 || nics > gpus) fail("nics_per_node out of range");
    const size_t want = static_cast<size_t>(nodes) * intra_per_node() + 2ull * nodes * nics +
                        static_cast<size_t>(nodes) * (nodes - 1) * nics;
    if (cap.size() != want || cls.size() != want || from.size() != want || to.size() != want)
        fail("unexpected link count");
    for (int i = 0; i < links(); ++i)
        if (!(cap[i] > 0)) fail("non-positive capacity on " + name(i));
    if (fabric == FabricKind::AllToAll) {
        for (int n = 0; n < nodes; ++n)
            for (int a = 0; a < gpus; ++a)
                for (int b = 0; b < gpus; ++b) {
                    if (a == b) continue;
                    const int id = mesh(n, a, b);
                    if (cls[id] != LinkClass::NvLink || from[id].index != a || to[id].index != b ||
                        from[id].node != n)
                        fail("NvLink index table broken");
                }
    } else {
        for (int n = 0; n < nodes; ++n)
            for (int g = 0; g < gpus; ++g)
                if (from[up(n, g)].index != g || to[down(n, g)].index != g) fail("port table broken");
    }
}

std::string shortest_double(double v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

// ---- line-oriented topology document (topology.cpp:296-403 format) ----

std::string save_link_model(const LinkModel& m) {
    std::string s;
    s += "nodes " + std::to_string(m.nodes) + "\n";
    s += "gpus_per_node " + std::to_string(m.gpus) + "\n";
    s += "nics_per_node " + std::to_string(m.nics) + "\n";
    s += std::string("fabric ") + (m.fabric == FabricKind::AllToAll ? "alltoall" : "nvswitch") + "\n";
    s += "nvlink_gbps " + shortest_double(m.nvlink_cap / 1e9) + "\n";
    if (m.rail_cap > 0) s += "rail_gbps " + shortest_double(m.rail_cap / 1e9) + "\n";
    for (int i = 0; i < m.links(); ++i) {
        const double dflt = m.cls[i] == LinkClass::Attach ? 2 * m.rail_cap
                            : m.cls[i] == LinkClass::Rail ? m.rail_cap
                                                          : m.nvlink_cap;
        if (m.cap[i] != dflt)
            s += "link " + endpoint_name(m.from[i]) + " " + endpoint_name(m.to[i]) + " " +
                 shortest_double(m.cap[i] / 1e9) + "\n";
    }
    return s;
}

namespace {

int to_int(const std::string& s, const char* what) {
    int v = 0;
    auto r = std::from_chars(s.data(), s.data() + s.size(), v);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size() || v < 0)
        throw std::runtime_error(std::string("bad ") + what + " '" + s + "'");
    return v;
}

Endpoint to_endpoint(const std::string& s) {
    auto bad = [&] { throw std::runtime_error("bad device name '" + s + "'"); };
    if (s.size() < 3 || s[0] != 'n') bad();
    const size_t dot = s.find('.');
    if (dot == std::string::npos || dot + 1 >= s.size()) bad();
    Endpoint e{to_int(s.substr(1, dot - 1), "node number"), kGpu, 0};
    const std::string rest = s.substr(dot + 1);
    if (rest == "sw") e.kind = kHub;
    else if (rest.size() > 3 && rest.compare(0, 3, "nic") == 0) e = {e.node, kNic, to_int(rest.substr(3), "nic index")};
    else if (rest.size() > 1 && rest[0] == 'g') e.index = to_int(rest.substr(1), "gpu index");
    else bad();
    return e;
}

}  // namespace

LinkModel load_link_model(const std::string& text) {
    int nodes = -1, gpus = -1, nics = -1;
    bool have_fabric = false;
    FabricKind fab = FabricKind::AllToAll;
    double nv = -1, rail = -1;
    struct Override { int line; std::string a, b, bw; };
    std::vector<Override> ov;
    std::istringstream in(text);
    std::string raw;
    int lineno = 0;
    auto die = [&](const std::string& msg) -> void {
        throw std::runtime_error("topology parse error at line " + std::to_string(lineno) + ": " + msg);
    };
    auto gb = [&](const std::string& s) {
        double v = 0;
        auto r = std::from_chars(s.data(), s.data() + s.size(), v);
        if (r.ec != std::errc() || r.ptr != s.data() + s.size()) die("bad number '" + s + "'");
        if (!(v > 0)) die("capacity must be positive, got '" + s + "'");
        return v;
    };
    while (std::getline(in, raw)) {
        ++lineno;
        if (auto h = raw.find('#'); h != std::string::npos) raw.resize(h);
        std::istringstream ls(raw);
        std::vector<std::string> tok;
        for (std::string t; ls >> t;) tok.push_back(t);
        if (tok.empty()) continue;
        const std::string& k = tok[0];
        auto arity = [&](size_t n) {
            if (tok.size() != n + 1) die("key '" + k + "' expects " + std::to_string(n) + " value(s)");
        };
        auto once = [&](bool seen) { if (seen) die("duplicate key '" + k + "'"); };
        if (k == "name") { arity(1); }
        else if (k == "nodes") { arity(1); once(nodes >= 0); nodes = to_int(tok[1], "nodes"); }
        else if (k == "gpus_per_node") { arity(1); once(gpus >= 0); gpus = to_int(tok[1], "gpus_per_node"); }
        else if (k == "nics_per_node") { arity(1); once(nics >= 0); nics = to_int(tok[1], "nics_per_node"); }
        else if (k == "fabric") {
            arity(1); once(have_fabric);
            if (tok[1] == "alltoall") fab = FabricKind::AllToAll;
            else if (tok[1] == "nvswitch") fab = FabricKind::NvSwitch;
            else die("fabric must be 'alltoall' or 'nvswitch', got '" + tok[1] + "'");
            have_fabric = true;
        } else if (k == "nvlink_gbps") { arity(1); once(nv >= 0); nv = gb(tok[1]); }
        else if (k == "rail_gbps") { arity(1); once(rail >= 0); rail = gb(tok[1]); }
        else if (k == "link") { arity(3); ov.push_back({lineno, tok[1], tok[2], tok[3]}); }
        else die("unknown key '" + k + "'");
    }
    auto need = [](bool ok, const char* what) {
        if (!ok) throw std::runtime_error(std::string("topology parse error: missing key '") + what + "'");
    };
    need(nodes >= 0, "nodes");
    need(gpus >= 0, "gpus_per_node");
    need(nics >= 0, "nics_per_node");
    need(have_fabric, "fabric");
    need(nv > 0, "nvlink_gbps");
    if (nics > 0) need(rail > 0, "rail_gbps");
    if (rail < 0) rail = 0;
    LinkModel m = make_link_model(nodes, gpus, nics, nv * 1e9, nics > 0 ? rail * 1e9 : 1.0, fab);
    if (nics == 0) m.rail_cap = rail * 1e9;
    for (const Override& o : ov) {
        lineno = o.line;
        Endpoint a{}, b{};
        try {
            a = to_endpoint(o.a);
            b = to_endpoint(o.b);
        } catch (const std::exception& e) {
            die(e.what());
        }
        const double bw = gb(o.bw) * 1e9;
        if (a.kind == kNic && b.kind == kNic && a.node != b.node && a.index != b.index)
            die("rail mismatch: " + o.a + " -> " + o.b + " (rails connect equal NIC indices)");
        const int id = m.find(a, b);
        if (id < 0) die("no such link " + o.a + " -> " + o.b);
        m.cap[id] = bw;
    }
    m.check();
    return m;
}

}  // namespace nb
