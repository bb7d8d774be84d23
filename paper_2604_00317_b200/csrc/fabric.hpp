// Link-load model: the directed, capacitated link index space the planner
// charges bytes against.  Semantics follow proj/include/nimble/topology.hpp and
// proj/src/topology.cpp:70-179 exactly (same dense link ids, same capacities),
// restated as flat arrays so the planner's inner loops index plain vectors.
//
//   NvSwitch fabric  (B200 HGX box): per GPU one up-port (GPU->switch) and one
//                    down-port (switch->GPU); ids [0,g) up, [g,2g) down per node.
//   AllToAll fabric  (NVLink mesh model): g(g-1) directed GPU->GPU links,
//                    id = src*(g-1) + (dst<src ? dst : dst-1) per node.
//   Then per node 2*nics GPU<->NIC attach links (2x rail rate), then rails over
//   ordered node pairs.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace nb {

enum class FabricKind : int { AllToAll = 0, NvSwitch = 1 };
enum class LinkClass : int { NvLink = 0, SwitchPort = 1, Attach = 2, Rail = 3 };

// Endpoint encoding: kind 0 = GPU, 1 = NIC, 2 = switch hub.
struct Endpoint {
    int node, kind, index;
    bool operator==(const Endpoint& o) const {
        return node == o.node && kind == o.kind && index == o.index;
    }
};

struct LinkModel {
    int nodes = 0, gpus = 0, nics = 0;
    FabricKind fabric = FabricKind::NvSwitch;
    double nvlink_cap = 0, rail_cap = 0;
    std::vector<double> cap;         // bytes/s per link id
    std::vector<LinkClass> cls;      // per link id
    std::vector<Endpoint> from, to;  // per link id

    int links() const { return static_cast<int>(cap.size()); }
    int intra_per_node() const {
        return fabric == FabricKind::AllToAll ? gpus * (gpus - 1) : 2 * gpus;
    }
    // dense-id formulas (topology.cpp:83-117); throw std::logic_error when absent
    int mesh(int node, int a, int b) const;
    int up(int node, int g) const;
    int down(int node, int g) const;
    int attach_up(int node, int nic) const;
    int attach_down(int node, int nic) const { return attach_up(node, nic) + 1; }
    int rail(int a, int b, int r) const;
    int find(const Endpoint& a, const Endpoint& b) const;
    std::string name(int id) const;
    void check() const;  // topology.cpp:181-252 invariants
};

LinkModel make_link_model(int nodes, int gpus, int nics, double nvlink_cap, double rail_cap,
                          FabricKind fabric);

std::string endpoint_name(const Endpoint& e);
std::string save_link_model(const LinkModel& m);
LinkModel load_link_model(const std::string& text);
std::string shortest_double(double v);

}  // namespace nb
