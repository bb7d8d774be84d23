// Traffic-matrix ingest: R x R byte demands, row = sender, zero diagonal.
// Generators restate proj/src/workloads.cpp:46-152 bit-exactly (the skewed
// hot share is a long-double product, the irregular matrix one mt19937_64
// stream); the payload-file format is workloads.cpp:154-198.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace nb {

struct Demand {
    int ranks = 0;
    std::vector<std::uint64_t> bytes;  // row-major

    std::uint64_t at(int s, int d) const { return bytes[static_cast<size_t>(s) * ranks + d]; }
    std::uint64_t& at(int s, int d) { return bytes[static_cast<size_t>(s) * ranks + d]; }
    void check() const;  // shape + zero diagonal (workloads.cpp:24-29)
};

Demand demand_p2p(int ranks, int src, int dst, std::uint64_t size);
Demand demand_skewed(int ranks, std::uint64_t per_rank, double ratio, int hot, bool per_sender_hot);
Demand demand_stencil(int ranks, std::uint64_t halo);
Demand demand_aggregator(int ranks, std::vector<int> dsts, std::uint64_t per_src);
Demand demand_irregular(int ranks, std::uint64_t total, double sparsity, std::uint64_t seed);

std::string demand_to_text(const Demand& m);
Demand demand_from_text(const std::string& text);

}  // namespace nb
