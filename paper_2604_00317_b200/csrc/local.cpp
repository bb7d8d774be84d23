// nimbleExchangeLocal: the 1-GPU emulated R-rank exchange (local-copy
// calibration of the forwarding engine).  One flagless engine launch moves
// every pair's segment; the same items, copy loops and grid as the NVLink
// path, with local addresses in place of peer ones.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>
#include <list>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nimble.h"
#include "capi_util.hpp"
#include "device.cuh"
#include "schedule.hpp"

namespace nb {
cudaError_t launch_exchange(const LaunchArgs& args, int ctas, cudaStream_t stream, bool pdl = true);
cudaError_t launch_gen(const GenArgs& g, cudaStream_t st);

namespace {

// A generated item list for one (matrix, buffers, chunk): the last few are
// kept, so alternating buffer sets (a pipelined caller) never rebuild.
struct LocalEntry {
    std::vector<uint64_t> key;
    Item* items = nullptr;
    size_t cap = 0, n = 0;
    cudaEvent_t used = nullptr;  // after the entry's last launch
};

constexpr size_t kLocalEntries = 4;

struct LocalCtx {
    bool ready = false;
    int sms = 148;
    CommDevice* d_view = nullptr;
    std::list<LocalEntry> entries;  // most recently used first
};

std::mutex g_mu;
std::map<int, LocalCtx> g_ctx;

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(nimbleUnhandledCudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

LocalCtx& context(int dev) {
    LocalCtx& c = g_ctx[dev];
    if (c.ready) return c;
    check(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev), "attribute");
    CommDevice v{};
    v.rank = 0;
    v.nranks = 1;
    check(cudaMalloc(&v.scratch, sizeof(uint32_t) * kScratchWords), "cudaMalloc");
    check(cudaMemset(v.scratch, 0, sizeof(uint32_t) * kScratchWords), "cudaMemset");
    check(cudaMalloc(&v.status, 64), "cudaMalloc");
    check(cudaMemset(v.status, 0, 64), "cudaMemset");
    check(cudaMalloc(&c.d_view, sizeof v), "cudaMalloc");
    check(cudaMemcpy(c.d_view, &v, sizeof v, cudaMemcpyHostToDevice), "cudaMemcpy");
    // the setup above ran on the legacy stream; launches may come on any stream
    check(cudaStreamSynchronize(cudaStreamLegacy), "cudaStreamSynchronize");
    c.ready = true;
    return c;
}

// The entry for `key`, generating its items on `st` when it is new: the
// flows go to the device generator as kernel parameters (or, beyond its
// capacity, are merged here and uploaded).  Reusing an old entry's buffer
// waits for its last launch on the stream, not on the host.
LocalEntry& entry_for(LocalCtx& c, const std::vector<uint64_t>& key, int R, const uint64_t* matrix,
                      const std::vector<uint64_t>& sb, const std::vector<uint64_t>& rb, uint64_t chunk,
                      cudaStream_t st) {
    for (auto it = c.entries.begin(); it != c.entries.end(); ++it)
        if (it->key == key) {
            c.entries.splice(c.entries.begin(), c.entries, it);
            return c.entries.front();
        }
    if (c.entries.size() >= kLocalEntries) {
        c.entries.splice(c.entries.begin(), c.entries, std::prev(c.entries.end()));
        check(cudaStreamWaitEvent(st, c.entries.front().used, 0), "cudaStreamWaitEvent");
    } else {
        c.entries.emplace_front();
        check(cudaEventCreateWithFlags(&c.entries.front().used, cudaEventDisableTiming), "cudaEventCreate");
    }
    LocalEntry& e = c.entries.front();
    e.key = key;
    std::vector<CutDesc> cuts = build_local_cuts(R, matrix, sb.data(), rb.data(), chunk);
    size_t n = 0;
    for (const CutDesc& f : cuts) n += f.n;
    if (n > e.cap) {
        if (e.items) check(cudaFreeAsync(e.items, st), "cudaFreeAsync");
        e.items = nullptr;
        check(cudaMallocAsync(reinterpret_cast<void**>(&e.items), n * sizeof(Item), st), "cudaMallocAsync");
        e.cap = n;
    }
    e.n = n;
    if (!n) return e;
    if (cuts.size() <= static_cast<size_t>(kMaxGenCuts)) {
        GenArgs g;
        std::memset(&g, 0, offsetof(GenArgs, cuts));
        g.items = e.items;
        g.ncuts = g.nkeyed = static_cast<uint32_t>(cuts.size());
        g.nitems = static_cast<uint32_t>(n);
        std::copy(cuts.begin(), cuts.end(), g.cuts);
        check(launch_gen(g, st), "schedule generation");
    } else {
        std::vector<Item> items = merge_cuts(cuts);
        check(cudaMemcpyAsync(e.items, items.data(), n * sizeof(Item), cudaMemcpyHostToDevice, st), "cudaMemcpy");
        check(cudaStreamSynchronize(st), "cudaStreamSynchronize");  // `items` is pageable and dies here
    }
    return e;
}

}  // namespace
}  // namespace nb

extern "C" nimbleResult_t nimbleExchangeLocal(int R, const void* const* sendbuffs, void* const* recvbuffs,
                                              const uint64_t* matrix, int ctas, void* stream) {
    return nb::guarded([&] {
        if (R < 1 || R > nb::kMaxRanks || !sendbuffs || !recvbuffs || !matrix)
            throw nb::Error(nimbleInvalidArgument, "local: bad argument");
        int dev = 0;
        nb::check(cudaGetDevice(&dev), "cudaGetDevice");
        std::lock_guard<std::mutex> lock(nb::g_mu);
        nb::LocalCtx& c = nb::context(dev);
        auto st = static_cast<cudaStream_t>(stream);
        const char* env = std::getenv("NIMBLE_LOCAL_CHUNK");
        const uint64_t chunk = env && *env ? std::strtoull(env, nullptr, 0) : (1ull << 20);
        std::vector<uint64_t> key(matrix, matrix + static_cast<size_t>(R) * R);
        std::vector<uint64_t> sb(R), rb(R);
        for (int r = 0; r < R; ++r) {
            sb[r] = reinterpret_cast<uint64_t>(sendbuffs[r]);
            rb[r] = reinterpret_cast<uint64_t>(recvbuffs[r]);
        }
        key.insert(key.end(), sb.begin(), sb.end());
        key.insert(key.end(), rb.begin(), rb.end());
        key.push_back(chunk);
        nb::LocalEntry& e = nb::entry_for(c, key, R, matrix, sb, rb, chunk, st);
        nb::LaunchArgs a{};
        a.items = e.items;
        a.nitems = static_cast<uint32_t>(e.n);
        a.slots = 1;
        a.pipe_chunk = chunk;
        a.comm = c.d_view;
        a.local_only = 1;
        int g = ctas > 0 ? ctas : c.sms;
        if (g > c.sms) g = c.sms;
        nb::check(nb::launch_exchange(a, g, st), "exchange launch");
        nb::check(cudaEventRecord(e.used, st), "cudaEventRecord");
    });
}
