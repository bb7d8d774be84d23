// Out-of-band rendezvous for one-process-per-GPU communicators: a TCP star on
// the host (loopback by default), the role NCCL's bootstrap network plays for
// ncclGetUniqueId / ncclCommInitRank.  Only small control blobs cross it
// (IPC handles at init and registration, demand-matrix rows when the planner
// needs the full matrix); no payload byte ever does.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "../../include/nimble.h"

namespace nb {

class Bootstrap {
  public:
    virtual ~Bootstrap() = default;
    // Every rank contributes `n` bytes; `all` receives nranks * n bytes in rank order.
    virtual void allgather(const void* mine, size_t n, void* all) = 0;
    void barrier() {
        uint8_t x = 0;
        std::vector<uint8_t> all(static_cast<size_t>(nranks));
        allgather(&x, 1, all.data());
    }
    int rank = 0, nranks = 1;
};

// Host shared memory between the ranks of one comm on one machine (POSIX
// shm, named after the comm's unique id): a lock-free allgather of small
// fixed-size records, for per-call metadata (the mesh model's demand-matrix
// rows) -- a few hundred nanoseconds instead of a TCP round trip through the
// bootstrap root.  Collective to create (uses the bootstrap's barrier).
class ShmAllgather {
  public:
    static constexpr size_t kRecord = 8 * 32;  // bytes per rank per call
    ShmAllgather(const nimbleUniqueId& id, Bootstrap& boot);
    ~ShmAllgather();
    // every rank contributes `n` <= kRecord bytes; `all` gets nranks * n bytes
    void allgather(const void* mine, size_t n, void* all, uint32_t timeout_ms);

  private:
    struct Slot;
    Slot* slots_ = nullptr;
    size_t bytes_ = 0;
    int rank_ = 0, nranks_ = 1;
    uint64_t calls_ = 0;
};

// Starts the root service in this process (detached thread) and describes how
// to reach it (address from NIMBLE_BOOTSTRAP_ADDR, default 127.0.0.1).
void bootstrap_root(nimbleUniqueId* id);
std::unique_ptr<Bootstrap> bootstrap_connect(const nimbleUniqueId& id, int rank, int nranks);

}  // namespace nb
