// nimbleExchangeLocal: the 1-GPU emulated R-rank exchange (local-copy
// calibration of the forwarding engine).  One flagless engine launch moves
// every pair's segment; the same items, copy loops and grid as the NVLink
// path, with local addresses in place of peer ones.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nimble.h"
#include "capi_util.hpp"
#include "device.cuh"
#include "schedule.hpp"

namespace nb {
cudaError_t launch_exchange(const LaunchArgs& args, int ctas, cudaStream_t stream);

namespace {

struct LocalCtx {
    bool ready = false;
    int sms = 148;
    CommDevice* d_view = nullptr;
    std::vector<uint64_t> key;
    Item* items = nullptr;
    size_t cap = 0, n = 0;
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
    check(cudaMalloc(&v.scratch, sizeof(uint32_t) * (2 + 2 * kMaxRanks)), "cudaMalloc");
    check(cudaMemset(v.scratch, 0, sizeof(uint32_t) * (2 + 2 * kMaxRanks)), "cudaMemset");
    check(cudaMalloc(&v.status, 64), "cudaMalloc");
    check(cudaMemset(v.status, 0, 64), "cudaMemset");
    check(cudaMalloc(&c.d_view, sizeof v), "cudaMalloc");
    check(cudaMemcpy(c.d_view, &v, sizeof v, cudaMemcpyHostToDevice), "cudaMemcpy");
    c.ready = true;
    return c;
}

}  // namespace
}  // namespace nb

extern "C" nimbleResult_t nimbleExchangeLocal(int R, const void* const* sendbuffs, void* const* recvbuffs,
                                              const uint64_t* matrix, int ctas, void* stream) {
    return nb::guarded([&] {
        if (R < 1 || !sendbuffs || !recvbuffs || !matrix) throw nb::Error(nimbleInvalidArgument, "local: bad argument");
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
        if (key != c.key) {
            std::vector<nb::Item> items = nb::build_local_items(R, matrix, sb.data(), rb.data(), chunk);
            nb::check(cudaStreamSynchronize(st), "cudaStreamSynchronize");  // previous launch may read the list
            if (items.size() > c.cap) {
                if (c.items) cudaFree(c.items);
                nb::check(cudaMalloc(&c.items, items.size() * sizeof(nb::Item)), "cudaMalloc");
                c.cap = items.size();
            }
            if (!items.empty())
                nb::check(cudaMemcpy(c.items, items.data(), items.size() * sizeof(nb::Item), cudaMemcpyHostToDevice),
                          "cudaMemcpy");
            c.n = items.size();
            c.key = key;
        }
        nb::LaunchArgs a{};
        a.items = c.items;
        a.nitems = static_cast<uint32_t>(c.n);
        a.slots = 1;
        a.pipe_chunk = chunk;
        a.comm = c.d_view;
        a.local_only = 1;
        int g = ctas > 0 ? ctas : c.sms;
        if (g > c.sms) g = c.sms;
        nb::check(nb::launch_exchange(a, g, st), "exchange launch");
    });
}
