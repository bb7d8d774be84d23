// C ABI, groups 2 and 3: communicator, registration, group semantics,
// send/recv / all-to-all(v), the 1-GPU emulated exchange and the bench entry
// points.  Host C++ around the sm_100a forwarding engine (engine.cu).
//
// Per call (stream-ordered, asynchronous, NCCL-style):
//   1. the group's ops become per-peer send / receive segments;
//   2. the planner runs on the comm's link-load model -- replicated on every
//      rank; the nvswitch model needs only this rank's row and column, the
//      mesh model gathers the full R x R matrix over the bootstrap;
//   3. the chunk scheduler turns plan + buffers into this rank's item list
//      (plan and schedule are cached, so a repeated exchange re-launches with
//      zero host work beyond the launch);
//   4. one forwarding-engine launch per rank.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nimble.h"
#include "bootstrap.hpp"
#include "capi_util.hpp"
#include "demand.hpp"
#include "device.cuh"
#include "fabric.hpp"
#include "planner.hpp"
#include "schedule.hpp"

namespace nb {
cudaError_t launch_exchange(const LaunchArgs& args, int ctas, cudaStream_t stream, bool pdl = true);
extern std::atomic<uint64_t> g_launch_seq;
cudaError_t launch_gen(const GenArgs& g, cudaStream_t st);
cudaError_t prepare_engine(int dev);
cudaError_t launch_fill(void* buf, uint64_t first, uint64_t n, uint64_t seed, int s, int d, cudaStream_t st);
cudaError_t launch_check(const void* buf, uint64_t first, uint64_t n, uint64_t seed, int s, int d, uint64_t* bad,
                         cudaStream_t st);
PlanParams to_params(const nimblePlannerConfig* c);
}  // namespace nb

#define CUDA_TRY(x)                                                                                            \
    do {                                                                                                       \
        cudaError_t e_ = (x);                                                                                  \
        if (e_ != cudaSuccess)                                                                                 \
            throw nb::Error(nimbleUnhandledCudaError, std::string(#x) + ": " + cudaGetErrorString(e_));       \
    } while (0)

namespace nb {
namespace {

using GetRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);

GetRangeFn address_range_fn() {
    static GetRangeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess)
            return static_cast<GetRangeFn>(nullptr);
        return reinterpret_cast<GetRangeFn>(p);
    }();
    return fn;
}

// allocation containing `ptr` (base, size)
std::pair<uint64_t, uint64_t> allocation_of(const void* ptr) {
    GetRangeFn fn = address_range_fn();
    if (!fn) throw Error(nimbleSystemError, "cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
        throw Error(nimbleInvalidArgument, "register: pointer is not device memory");
    return {base, size};
}

uint64_t fnv(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
    auto* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

size_t elem_size(nimbleDataType_t t) {
    switch (t) {
    case nimbleInt8:
    case nimbleUint8:
    case nimbleFloat8e4m3:
    case nimbleFloat8e5m2: return 1;
    case nimbleFloat16:
    case nimbleBfloat16: return 2;
    case nimbleInt32:
    case nimbleUint32:
    case nimbleFloat32: return 4;
    case nimbleInt64:
    case nimbleUint64:
    case nimbleFloat64: return 8;
    default: throw Error(nimbleInvalidArgument, "bad datatype");
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) CUDA_TRY(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// One internal stream per device for the library's own host -> device state
// writes and stream-ordered frees, created once per process and never
// destroyed.  A device offers a fixed number of hardware work queues (32
// connections at most); every stream created maps onto one, round robin.  On
// a device hosting several ranks of a comm, a stream that shares a queue
// with a peer rank's spinning engine waits behind it -- so the library
// creates no stream per comm (streams created and destroyed with every comm
// keep shifting which queues collide).
cudaStream_t internal_stream(int dev) {
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    if (dev < 0 || dev >= 64) throw Error(nimbleInvalidArgument, "device index out of range");
    std::lock_guard<std::mutex> g(mu);
    if (!streams[dev]) CUDA_TRY(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
    return streams[dev];
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n;
            o.p = nullptr, o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    // Stream-ordered (de)allocation from the comm's pool: cudaFree would
    // synchronize the whole device, and on a device hosting several ranks of
    // one comm that means waiting for a peer's engine grid that may itself
    // wait for this rank's next launch.  The buffer is idle whenever it grows
    // or is released (the schedule cache orders it after the entry's last
    // launch first).  Capacity grows by powers of two.
    void reserve(size_t m, cudaStream_t st, cudaMemPool_t pool) {
        if (m <= n && p) return;
        if (p) CUDA_TRY(cudaFreeAsync(p, st));
        p = nullptr;
        size_t cap = 64;
        while (cap < m) cap *= 2;
        CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), cap * sizeof(T), pool, st));
        n = cap;
    }
    void assign(const std::vector<T>& v, cudaStream_t st, cudaMemPool_t pool) {
        reserve(v.size(), st, pool);
        if (!v.empty()) CUDA_TRY(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    }
    void release() {
        int dev = 0;
        if (p && cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) cudaFreeAsync(p, internal_stream(dev));
        else if (p) cudaFreeAsync(p, cudaStreamPerThread);
        p = nullptr;
        n = 0;
    }
};

struct PeerInfo {
    int32_t pid;
    int32_t dev;
    uint64_t host;
    uint64_t ctrl_ptr, staging_ptr;  // raw pointers: a peer in this process maps nothing
    cudaIpcMemHandle_t ctrl, staging;
};

struct Window {
    bool live = false;
    uint64_t base = 0, size = 0;  // registered range (local)
    std::vector<void*> opened;    // IPC mappings to close
};

struct CachedPlan {
    std::vector<uint64_t> key;
    std::shared_ptr<PlanResult> plan;
    uint64_t id = 0;
    double seconds = 0;
};

// Pin count of a schedule captured into CUDA graphs: shared with the graphs'
// user objects, whose destructors (CUDA-internal threads, no CUDA calls
// allowed) only decrement it.
struct GraphPins {
    std::atomic<int> n{0};
};

struct CachedSchedule {
    std::vector<uint64_t> key;
    Schedule sc;
    DevBuf<Item> items;
    DevBuf<Post> posts;
    DevBuf<Post> send_posts;
    DevBuf<uint64_t> finals;
    DevBuf<Item> ll_items;
    cudaEvent_t used = nullptr;  // recorded after every eager launch of this entry
    std::shared_ptr<GraphPins> pins = std::make_shared<GraphPins>();
    CachedSchedule() = default;
    CachedSchedule(const CachedSchedule&) = delete;
    CachedSchedule(CachedSchedule&& o) noexcept
        : key(std::move(o.key)), sc(std::move(o.sc)), items(std::move(o.items)), posts(std::move(o.posts)),
          send_posts(std::move(o.send_posts)), finals(std::move(o.finals)), ll_items(std::move(o.ll_items)),
          used(o.used), pins(std::move(o.pins)) {
        o.used = nullptr;
    }
    ~CachedSchedule() {
        if (used) cudaEventDestroy(used);
    }
    bool pinned() const { return pins && pins->n.load() > 0; }
    // no launch of this comm still reads the entry's device buffers
    void wait_idle() const {
        if (used) cudaEventSynchronize(used);
    }
};

struct Clique;

// Process-wide cache of opened IPC handles: one allocation may back several
// registered windows, and a handle may be opened only once per process.
struct IpcCache {
    std::mutex m;
    std::map<std::string, std::pair<void*, int>> open;  // handle bytes -> (base, refs)
    void* acquire(const cudaIpcMemHandle_t& h) {
        std::lock_guard<std::mutex> g(m);
        std::string k(reinterpret_cast<const char*>(&h), sizeof h);
        auto it = open.find(k);
        if (it != open.end()) {
            ++it->second.second;
            return it->second.first;
        }
        void* p = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        open[k] = {p, 1};
        return p;
    }
    void release(void* p) {
        std::lock_guard<std::mutex> g(m);
        for (auto it = open.begin(); it != open.end(); ++it)
            if (it->second.first == p) {
                if (--it->second.second == 0) {
                    cudaIpcCloseMemHandle(p);
                    open.erase(it);
                }
                return;
            }
    }
};

IpcCache& ipc_cache() {
    static IpcCache c;
    return c;
}

}  // namespace
}  // namespace nb

struct nimbleComm {
    int rank = 0, nranks = 1, device = 0, sms = 148;
    // ranks of this comm on my device (one process, several streams): their
    // engine grids must all be resident at once, so each launch takes at most
    // sms_share CTAs by default
    int colocated = 1, sms_share = 148;
    std::unique_ptr<nb::Bootstrap> boot;
    std::unique_ptr<nb::ShmAllgather> shm;  // per-call metadata between ranks (mesh model rows)
    std::shared_ptr<nb::Clique> clique;
    nimbleCommConfig cfg{};
    uint8_t* ctrl = nullptr;
    uint8_t* staging = nullptr;
    uint64_t staging_bytes = 0;
    std::vector<uint8_t*> peer_ctrl, peer_staging;
    std::vector<void*> ipc_mapped;  // ctrl / staging mappings of peers
    nb::CommDevice view{};
    nb::CommDevice view_on_device{};  // what d_view holds (upload_view skips identical writes)
    bool view_uploaded = false;
    nb::CommDevice* d_view = nullptr;
    uint64_t* d_win_table = nullptr;
    uint64_t* d_epoch = nullptr;
    uint32_t* d_scratch = nullptr;
    uint32_t* h_status = nullptr;  // host-mapped async error word
    uint32_t* d_status = nullptr;  // its device alias
    std::vector<nb::Window> windows;
    std::vector<uint64_t> win_table;  // [win * kMaxRanks + rank]
    uint64_t plan_ids = 0;
    std::list<nb::CachedPlan> plans;
    std::list<nb::CachedSchedule> schedules;
    std::list<nb::CachedSchedule> retired;  // evicted while pinned by a CUDA graph
    // Repeat fast path: the previous stand-alone all-to-allv (buffers, counts;
    // nvswitch model) and the cached schedule it launched.  Cleared whenever
    // schedules, windows or the config change.
    struct {
        nb::CachedSchedule* cs = nullptr;
        nb::RankBuffers rb;
        uint64_t key[2 + 4 * nb::kMaxRanks];
    } fast;
    nb::CachedSchedule* last_cs = nullptr;  // schedule of the most recent launch
    nb::RankBuffers last_rb;
    cudaStream_t bench_stream = nullptr;
    // host -> device updates of the comm's own state (view, window table,
    // flags at init): an internal non-blocking stream, synchronized before the
    // call returns -- the legacy stream would not order them before a peer
    // rank's kernels on other streams (ranks sharing a device)
    cudaStream_t aux = nullptr;
    cudaMemPool_t pool = nullptr;  // schedule buffers (DevBuf)
    uint64_t* d_trace = nullptr;  // NIMBLE_TRACE=1: device timeline of the last launch
    nb::DeviceStats* d_stats = nullptr;  // NIMBLE_STATS=1: per-kind byte counters, slot occupancy
    struct {
        uint64_t calls = 0, ns = 0, ns_max = 0, plans = 0, plan_ns = 0, schedules = 0, schedule_ns = 0;
        uint64_t launches = 0;
    } host;  // C ABI cost per data-path call (nimbleCommGetStats)
    cudaEvent_t last_launch = nullptr;  // launches on one comm are serialized across streams
    cudaStream_t last_stream = nullptr;
    bool launched = false;
    // Epoch chaining (LaunchArgs::prev_epoch): the host's count of this comm's
    // launches -- exact until a launch is captured into a CUDA graph (replays
    // advance the device epoch unseen) -- and the library launch counter and
    // stream right after the previous exchange.
    uint64_t host_epoch = 0;
    bool epoch_known = true;
    uint64_t chain_seq = ~0ull;
    cudaStream_t chain_stream = nullptr;
    // Frees whatever device / host state exists, so a comm whose init failed
    // half-way releases what it had allocated (nimbleCommDestroy first makes
    // sure no peer still touches it).
    ~nimbleComm();
};

namespace nb {
namespace {

struct Clique {
    std::vector<nimbleComm*> comms;
    struct Region {
        int device;
        uint8_t* ctrl;
        uint8_t* staging;
    };
    std::vector<Region> deferred;  // ctrl / staging of destroyed members
    ~Clique() {
        int prev = -1;
        cudaGetDevice(&prev);
        for (const Region& r : deferred) {
            if (cudaSetDevice(r.device) != cudaSuccess) continue;
            cudaDeviceSynchronize();
            cudaFree(r.ctrl);
            cudaFree(r.staging);
        }
        cudaGetLastError();
        if (prev >= 0) cudaSetDevice(prev);
    }
};

uint64_t ring_count(const nimbleComm* c, const nimbleCommConfig& cfg);

// Complete host -> device writes of comm state (see nimbleComm::aux).
void h2d(nimbleComm* c, void* dst, const void* src, size_t n) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, c->aux));
    CUDA_TRY(cudaStreamSynchronize(c->aux));
}

void zero(nimbleComm* c, void* dst, size_t n) {
    CUDA_TRY(cudaMemsetAsync(dst, 0, n, c->aux));
    CUDA_TRY(cudaStreamSynchronize(c->aux));
}

void upload_view(nimbleComm* c) {
    c->view.rank = c->rank;
    c->view.nranks = c->nranks;
    for (int r = 0; r < c->nranks; ++r) {
        c->view.ctrl[r] = c->peer_ctrl[static_cast<size_t>(r)];
        c->view.staging[r] = c->peer_staging[static_cast<size_t>(r)];
    }
    c->view.win_table = c->d_win_table;
    c->view.nwin = static_cast<uint32_t>(c->windows.size());
    c->view.status = c->d_status;
    c->view.scratch = c->d_scratch;
    c->view.stats = c->d_stats;
    c->view.ring_full = ring_count(c, c->cfg) > static_cast<uint64_t>(c->nranks) ? 1u : 0u;
    c->view.epoch = c->d_epoch;
    const char* t = std::getenv("NIMBLE_TIMEOUT_MS");
    c->view.timeout_ms = t && *t ? static_cast<uint32_t>(std::atoi(t)) : 60000u;
    // Only when it changed: a config change that is host-side only (pull
    // mode, chunk sizes of direct items, LL limit) then touches no device
    // memory -- no stream operation that could queue behind a co-resident
    // peer's running engine (see internal_stream).
    if (c->view_uploaded && std::memcmp(&c->view_on_device, &c->view, sizeof c->view) == 0) return;
    h2d(c, c->d_view, &c->view, sizeof c->view);
    c->view_on_device = c->view;
    c->view_uploaded = true;
}

constexpr uint32_t kMaxWindows = 256;
constexpr uint64_t kDefaultDirectChunk = 128ull << 10;
// Direct pushes default to 8 KiB items: on 4 B200s the skewed exchange's hot
// port (pulling in, pushing out) gains 0.03-0.09 of the bound at hotspot
// ratios 0.6-0.8 over 64 KiB, and push-only traffic does not lose
// (profiles/r01_push_chunk.md).
constexpr uint64_t kDefaultPushChunk = 8ull << 10;

uint32_t slot_count(const nimbleCommConfig& cfg) {
    if (cfg.pipe_chunk == 0) throw Error(nimbleInvalidArgument, "config: pipe_chunk must be positive");
    const uint64_t s = static_cast<uint64_t>(cfg.channels_per_peer) * (cfg.p2p_buffer / cfg.pipe_chunk);
    if (s == 0) throw Error(nimbleInvalidArgument, "config: p2p_buffer holds less than one chunk");
    if (s > kMaxSlots) throw Error(nimbleInvalidArgument, "config: more than 256 staging slots per ring");
    return static_cast<uint32_t>(s);
}

// Staging rings hosted per rank.  Under the nvswitch model the planner never
// relays, so a rank hosts only its self rings -- one per sender, fed by
// pushes into an unregistered receive buffer: R rings (80 MiB at R = 8 with
// the 10 MiB reference geometry).  The mesh model may route any pair through
// any rank: R x R rings (ring (s, d) at index s * R + d).
uint64_t ring_count(const nimbleComm* c, const nimbleCommConfig& cfg) {
    const uint64_t R = static_cast<uint64_t>(c->nranks);
    return cfg.fabric == nimbleFabricAllToAll ? R * R : R;
}

uint64_t staging_size(const nimbleComm* c) {
    return ring_count(c, c->cfg) * slot_count(c->cfg) * c->cfg.pipe_chunk;
}

// Hash of the data-path geometry every rank must share: where chunks land in
// rings and slots, how pairs are cut, which pairs ride LL, which model plans.
uint64_t geometry_hash(const nimbleCommConfig& cfg) {
    const uint64_t v[] = {cfg.pipe_chunk, cfg.p2p_buffer, static_cast<uint64_t>(cfg.channels_per_peer),
                          cfg.push_chunk, cfg.direct_chunk, cfg.ll_max, static_cast<uint64_t>(cfg.fabric),
                          static_cast<uint64_t>(cfg.gpus_per_node)};
    return fnv(v, sizeof v);
}

void default_config(nimbleCommConfig* cfg, int nranks) {
    std::memset(cfg, 0, sizeof *cfg);
    cfg->fabric = nimbleFabricNvSwitch;
    cfg->gpus_per_node = nranks;
    cfg->nvlink_bytes_per_s = 900e9;
    nimblePlannerConfigDefault(&cfg->planner);
    // Same 10 MiB per ring as the reference's PipelineConfig (pipeline.hpp:18),
    // cut finer: 160 x 64 KiB slots keep ~160 CTAs busy on one relayed flow
    // (20 x 512 KiB capped it at 20).
    cfg->pipe_chunk = 64ull << 10;
    cfg->p2p_buffer = 10ull << 20;
    cfg->channels_per_peer = 1;
    cfg->ctas = 0;
    cfg->direct_chunk = 0;
    cfg->pull = 0;
    cfg->push_chunk = 0;
    cfg->ll_max = kLLMaxData;
}

// Peer access from the current device to `dev` (idempotent).
void enable_peer(int dev) {
    cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else CUDA_TRY(e);
}

// Default CTAs per launch.  A device hosting k ranks of this comm (one
// process, k streams) runs k engine grids at once, and each grid's producers
// spin on flags raised by the others: all of them must be resident together,
// and the kernels each rank runs between its exchanges (on its own stream,
// possibly with large shared-memory footprints) must still find SMs while
// the other ranks' grids spin.  So each grid takes SMs / 2k CTAs, and the
// grids are launched without programmatic dependent launch (a grid whose
// successor is pre-launched would hold twice its share).
//
// CUDA loads a kernel's module on the kernel's first launch (lazy loading,
// the default), and a module load waits for the device's running kernels:
// here, the peer ranks' grids, which spin until this rank's next exchange --
// a kernel first used between two exchanges stalls every rank until the
// engine's timeout (tools/first_use_probe.py).  The library loads its own
// kernels at comm creation (prepare_engine); the process's other kernels
// need CUDA_MODULE_LOADING=EAGER, said once on stderr.
void set_share(nimbleComm* c) {
    c->sms_share = c->colocated <= 1 ? c->sms : std::max(1, c->sms / (2 * c->colocated));
    static std::atomic<bool> warned{false};
    const char* mode = std::getenv("CUDA_MODULE_LOADING");
    if (c->colocated > 1 && !(mode && std::strcmp(mode, "EAGER") == 0) && !warned.exchange(true))
        std::fprintf(stderr,
                     "nimble: %d ranks of one comm share GPU %d and CUDA_MODULE_LOADING is not EAGER: a kernel "
                     "loaded lazily between two exchanges waits for the peer ranks' running engines "
                     "(set CUDA_MODULE_LOADING=EAGER before CUDA initializes)\n",
                     c->colocated, c->device);
}

// Allocate ctrl + staging, exchange handles / pointers, map peers.
void setup_regions(nimbleComm* c, bool single_process) {
    DeviceGuard g(c->device);
    c->staging_bytes = staging_size(c);
    const uint64_t ctrl_bytes = FlagLayout::bytes(c->nranks);
    CUDA_TRY(cudaMalloc(&c->ctrl, ctrl_bytes));
    zero(c, c->ctrl, ctrl_bytes);
    CUDA_TRY(cudaMalloc(&c->staging, std::max<uint64_t>(c->staging_bytes, 256)));
    c->peer_ctrl.assign(static_cast<size_t>(c->nranks), nullptr);
    c->peer_staging.assign(static_cast<size_t>(c->nranks), nullptr);
    c->peer_ctrl[static_cast<size_t>(c->rank)] = c->ctrl;
    c->peer_staging[static_cast<size_t>(c->rank)] = c->staging;
    if (single_process) return;  // the clique fills peers in directly
    PeerInfo mine{};
    mine.pid = ::getpid();
    mine.dev = c->device;
    mine.host = ::gethostid();
    mine.ctrl_ptr = reinterpret_cast<uint64_t>(c->ctrl);
    mine.staging_ptr = reinterpret_cast<uint64_t>(c->staging);
    CUDA_TRY(cudaIpcGetMemHandle(&mine.ctrl, c->ctrl));
    CUDA_TRY(cudaIpcGetMemHandle(&mine.staging, c->staging));
    std::vector<PeerInfo> all(static_cast<size_t>(c->nranks));
    c->boot->allgather(&mine, sizeof mine, all.data());
    c->colocated = 0;
    for (int r = 0; r < c->nranks; ++r) {
        const PeerInfo& p = all[static_cast<size_t>(r)];
        if (p.host != mine.host) throw Error(nimbleInvalidUsage, "comm: ranks must share one NVLink box");
        if (p.dev == mine.dev) {
            // ranks sharing a device must share a process (streams of one
            // context run concurrently; separate processes time-slice, and
            // the engines' flag waits would stall)
            if (p.pid != mine.pid)
                throw Error(nimbleInvalidUsage, "comm: ranks on one GPU must live in one process (one thread each)");
            ++c->colocated;
        }
    }
    for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) continue;
        const PeerInfo& p = all[static_cast<size_t>(r)];
        if (p.pid == mine.pid) {
            // a rank of this process (one thread per rank): its pointers are
            // valid here as they are, given peer access to its device
            if (p.dev != mine.dev) enable_peer(p.dev);
            c->peer_ctrl[static_cast<size_t>(r)] = reinterpret_cast<uint8_t*>(p.ctrl_ptr);
            c->peer_staging[static_cast<size_t>(r)] = reinterpret_cast<uint8_t*>(p.staging_ptr);
            continue;
        }
        void* a = nullptr;
        void* b = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&a, p.ctrl, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_mapped.push_back(a);
        CUDA_TRY(cudaIpcOpenMemHandle(&b, p.staging, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_mapped.push_back(b);
        c->peer_ctrl[static_cast<size_t>(r)] = static_cast<uint8_t*>(a);
        c->peer_staging[static_cast<size_t>(r)] = static_cast<uint8_t*>(b);
    }
    set_share(c);
}

void setup_common(nimbleComm* c) {
    DeviceGuard g(c->device);
    CUDA_TRY(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
    CUDA_TRY(prepare_engine(c->device));
    c->aux = internal_stream(c->device);
    // The comm's own memory pool for schedule buffers, which grow while
    // other ranks' engines may be running: it keeps what it maps (release
    // threshold: never) and starts with room for ~500k work items, so a new
    // schedule normally allocates without touching the device's mappings.
    {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = c->device;
        CUDA_TRY(cudaMemPoolCreate(&c->pool, &props));
        uint64_t keep = ~0ull;
        CUDA_TRY(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
        // No allocation may wait on another stream's pending free (the
        // allocator's "internal dependencies"): on a device hosting several
        // ranks, the stream holding that free can share a hardware queue with
        // a peer's spinning engine (see internal_stream).  Freed blocks are
        // reused once their frees have completed.
        int no = 0;
        CUDA_TRY(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &no));
        void* warm = nullptr;
        CUDA_TRY(cudaMallocFromPoolAsync(&warm, 16ull << 20, c->pool, c->aux));
        CUDA_TRY(cudaFreeAsync(warm, c->aux));
        CUDA_TRY(cudaStreamSynchronize(c->aux));
    }
    CUDA_TRY(cudaMalloc(&c->d_view, sizeof(CommDevice)));
    CUDA_TRY(cudaMalloc(&c->d_win_table, sizeof(uint64_t) * kMaxWindows * kMaxRanks));
    zero(c, c->d_win_table, sizeof(uint64_t) * kMaxWindows * kMaxRanks);
    CUDA_TRY(cudaMalloc(&c->d_epoch, sizeof(uint64_t)));
    zero(c, c->d_epoch, sizeof(uint64_t));
    CUDA_TRY(cudaMalloc(&c->d_scratch, sizeof(uint32_t) * kScratchWords));
    zero(c, c->d_scratch, sizeof(uint32_t) * kScratchWords);
    CUDA_TRY(cudaHostAlloc(&c->h_status, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(c->h_status, 0, 64);
    CUDA_TRY(cudaHostGetDevicePointer(&c->d_status, c->h_status, 0));
    CUDA_TRY(cudaEventCreateWithFlags(&c->last_launch, cudaEventDisableTiming));
    if (const char* t = std::getenv("NIMBLE_TRACE"); t && *t == '1') {
        CUDA_TRY(cudaMalloc(&c->d_trace, sizeof(uint64_t) * kTraceRegionWords));
        std::vector<uint64_t> init(kTraceRegionWords, 0);
        for (int b = 0; b < 2; ++b)
            for (int k = 0; k < kTraceSlots; ++k)
                if (trace_is_min_slot(k)) init[static_cast<size_t>(b * kTraceWords + k)] = ~0ull;
        h2d(c, c->d_trace, init.data(), init.size() * sizeof(uint64_t));
    }
    if (const char* t = std::getenv("NIMBLE_STATS"); t && *t == '1') {
        CUDA_TRY(cudaMalloc(&c->d_stats, sizeof(DeviceStats)));
        zero(c, c->d_stats, sizeof(DeviceStats));
    }
    c->win_table.assign(static_cast<size_t>(kMaxWindows) * kMaxRanks, 0);
}

// Never throws; the caller has made c's device current.
void free_regions(nimbleComm* c) {
    for (void* p : c->ipc_mapped) cudaIpcCloseMemHandle(p);
    c->ipc_mapped.clear();
    if (c->ctrl) cudaFree(c->ctrl);
    if (c->staging) cudaFree(c->staging);
    c->ctrl = c->staging = nullptr;
}

// Wait until no launch of this comm is in flight.  A device hosting one rank
// syncs the device (graph replays included).  A device hosting several ranks
// of the comm waits for this comm's last eager launch only: a device-wide
// sync there would also wait for peer grids that may be waiting for this
// rank's next launch (graph replays must be synchronized by the caller).
void quiesce(nimbleComm* c) {
    if (c->colocated > 1) {
        if (c->launched) CUDA_TRY(cudaEventSynchronize(c->last_launch));
    } else {
        CUDA_TRY(cudaDeviceSynchronize());
    }
}

// ---------------------------------------------------------------- planning

LinkModel comm_model(const nimbleComm* c) {
    const int gpn = std::max(c->cfg.gpus_per_node, c->nranks);
    const FabricKind f = c->cfg.fabric == nimbleFabricAllToAll ? FabricKind::AllToAll : FabricKind::NvSwitch;
    return make_link_model(1, gpn, 0, c->cfg.nvlink_bytes_per_s, 0.0, f);
}

std::shared_ptr<PlanResult> plan_for(nimbleComm* c, const std::vector<uint64_t>& matrix, uint64_t* plan_id) {
    std::vector<uint64_t> key = matrix;
    key.push_back(fnv(&c->cfg, sizeof c->cfg));
    for (auto it = c->plans.begin(); it != c->plans.end(); ++it)
        if (it->key == key) {
            c->plans.splice(c->plans.begin(), c->plans, it);
            *plan_id = it->id;
            return it->plan;
        }
    const auto t0 = std::chrono::steady_clock::now();
    const LinkModel lm = comm_model(c);
    Demand d;
    d.ranks = c->nranks;
    d.bytes = matrix;
    struct Timed {
        nimbleComm* c;
        std::chrono::steady_clock::time_point t0;
        ~Timed() {
            ++c->host.plans;
            c->host.plan_ns += static_cast<uint64_t>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
        }
    } timed{c, t0};
    // On the nvswitch model every pair has exactly one candidate (direct), so
    // the MCF sweep can only put each pair's demand on it: the direct plan has
    // the same flows (tests/test_planner_parity.py) at a fraction of the cost
    // -- it matters when every call brings a new matrix (MoE dispatch).
    auto p = std::make_shared<PlanResult>(c->cfg.fabric == nimbleFabricNvSwitch
                                              ? direct_plan(lm, c->nranks, lm.gpus, d)
                                              : mcf_plan(lm, c->nranks, lm.gpus, d, to_params(&c->cfg.planner)));
    c->plans.push_front({key, p, ++c->plan_ids, p->stats.wall_seconds});
    if (c->plans.size() > 4) c->plans.pop_back();
    *plan_id = c->plan_ids;
    return p;
}

// ---------------------------------------------------------------- groups

struct PendingOp {
    enum Kind { Send, Recv, AllToAllV } kind;
    nimbleComm* comm;
    cudaStream_t stream;
    int peer;
    uint64_t ptr, bytes;                                      // Send / Recv
    uint64_t sbase, rbase;                                    // AllToAllV
    std::vector<uint64_t> sbytes, soff, rbytes, roff;         // AllToAllV (bytes)
};

thread_local int g_group_depth = 0;
thread_local std::vector<PendingOp> g_pending;

struct Exchange {
    nimbleComm* comm;
    cudaStream_t stream;
    std::vector<cudaStream_t> others;
    RankBuffers rb;
    std::vector<bool> has_send, has_recv;
};

Exchange make_exchange(nimbleComm* c, const std::vector<PendingOp*>& ops) {
    Exchange ex;
    ex.comm = c;
    ex.stream = ops.front()->stream;
    const int R = c->nranks;
    ex.rb.R = R;
    ex.rb.me = c->rank;
    ex.rb.send_ptr.assign(R, 0);
    ex.rb.send_bytes.assign(R, 0);
    ex.rb.recv_ptr.assign(R, 0);
    ex.rb.recv_bytes.assign(R, 0);
    ex.has_send.assign(R, false);
    ex.has_recv.assign(R, false);
    // NCCL group semantics: several sends to (receives from) one peer are
    // matched in issue order with the peer's receives (sends); the pair then
    // consists of those parts, in that order
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> sends(static_cast<size_t>(R)), recvs(static_cast<size_t>(R));
    for (PendingOp* op : ops) {
        if (op->stream != ex.stream &&
            std::find(ex.others.begin(), ex.others.end(), op->stream) == ex.others.end())
            ex.others.push_back(op->stream);
        if (op->kind == PendingOp::Send) sends[static_cast<size_t>(op->peer)].push_back({op->ptr, op->bytes});
        else if (op->kind == PendingOp::Recv) recvs[static_cast<size_t>(op->peer)].push_back({op->ptr, op->bytes});
        else
            for (int p = 0; p < R; ++p) {
                sends[static_cast<size_t>(p)].push_back({op->sbase + op->soff[p], op->sbytes[p]});
                recvs[static_cast<size_t>(p)].push_back({op->rbase + op->roff[p], op->rbytes[p]});
            }
    }
    auto settle = [&](std::vector<std::pair<uint64_t, uint64_t>>& parts, std::vector<bool>& has,
                      std::vector<uint64_t>& ptr, std::vector<uint64_t>& bytes,
                      std::vector<std::vector<std::pair<uint64_t, uint64_t>>>& multi, int p) {
        if (parts.empty()) return;
        has[static_cast<size_t>(p)] = true;
        if (parts.size() > 1)  // zero-byte operations carry nothing (both ends drop them alike)
            parts.erase(std::remove_if(parts.begin(), parts.end(), [](const auto& x) { return x.second == 0; }),
                        parts.end());
        if (parts.empty()) return;
        ptr[static_cast<size_t>(p)] = parts[0].first;
        uint64_t total = 0;
        for (const auto& x : parts) total += x.second;
        bytes[static_cast<size_t>(p)] = total;
        if (parts.size() > 1) {
            if (p == c->rank) throw Error(nimbleInvalidUsage, "group: several operations on the self segment");
            if (multi.empty()) multi.resize(static_cast<size_t>(R));
            multi[static_cast<size_t>(p)] = parts;
        }
    };
    for (int p = 0; p < R; ++p) {
        settle(sends[static_cast<size_t>(p)], ex.has_send, ex.rb.send_ptr, ex.rb.send_bytes, ex.rb.send_parts, p);
        settle(recvs[static_cast<size_t>(p)], ex.has_recv, ex.rb.recv_ptr, ex.rb.recv_bytes, ex.rb.recv_parts, p);
    }
    if ((!ex.rb.send_parts.empty() || !ex.rb.recv_parts.empty()) && c->cfg.fabric == nimbleFabricAllToAll)
        throw Error(nimbleInvalidUsage, "group: several operations per peer need the nvswitch model");
    return ex;
}

// Registered window holding [ptr, ptr + n), or -1.
int window_of(const nimbleComm* c, uint64_t ptr, uint64_t n) {
    for (size_t w = 0; w < c->windows.size(); ++w) {
        const Window& win = c->windows[w];
        if (win.live && ptr >= win.base && ptr + n <= win.base + win.size) return static_cast<int>(w);
    }
    return -1;
}

// NIMBLE_PUSH_DISTANCES=mask (experiment, 0 = off): receivers do not ask
// senders at ring distance d (me - s mod R) with bit d set to be pulled from,
// so those pairs are pushed -- a per-pair push / pull split of balanced ports.
uint64_t push_distances() {
    static const uint64_t m = [] {
        const char* e = std::getenv("NIMBLE_PUSH_DISTANCES");
        return static_cast<uint64_t>(e && *e ? std::strtoull(e, nullptr, 0) : 0);
    }();
    return m;
}

// Where each incoming segment lands: a registered window (zero copy) or the
// self ring (staged); where each outgoing segment lives (registered windows
// can be pulled by their receiver); whether this rank asks to pull.
void fill_posts(nimbleComm* c, RankBuffers& rb, const PlanResult& plan) {
    for (int p = 0; p < rb.R; ++p)
        if (rb.send_bytes[p] >> 48 || rb.recv_bytes[p] >> 48 || rb.recv_ptr[p] >> 48)
            throw Error(nimbleInvalidArgument, "alltoallv: segments must be < 2^48 bytes and addresses < 2^48");
    uint64_t ingress = 0, egress = 0;
    for (int p = 0; p < rb.R; ++p)
        if (p != rb.me) ingress += rb.recv_bytes[p], egress += rb.send_bytes[p];
    // Push or pull, per port, from this rank's own row and column (measured on
    // 2-4 B200s, profiles/r01_summary.md, r01_pull_policy.md):
    //  - a pull loads the *sender's* ingress with read requests (24 B per
    //    128 B); a push loads the receiver's egress with almost nothing;
    //  - pull responses carry 16 B of protocol per 128 B, writes 24 B;
    //  - mixing pushes and pulls on links busy both ways is slow.
    // Receivers always ask to pull; a sender declines -- and pushes its data
    // out -- only when its own port is clearly ingress-bound, so the hot port
    // of a skewed exchange pulls everything in and pushes everything out.
    // "Clearly": ingress > 1.2 x egress with three or more ranks, > 1.55 x with
    // two.  A decliner drives both directions from its own engine (~1.08 TB/s
    // of pushes plus pulls on one B200) while its peers' engines lose that
    // work; with a single peer nothing else is left for the peer to do, so
    // declining pays only at a larger imbalance (profiles/r01_pull_policy.md,
    // threshold study on 2-4 GPUs with 8 KiB pushes).
    // Two ranks whose directions are within 1.5x of each other both push: with
    // every byte crossing the one link pair in both directions, pull requests
    // ride on the other direction's data and two-way pushes come out ahead
    // (0.75 vs 0.72-0.74 of the bound at r >= 0.7 and for uniform traffic).
    // Each rank's row and column are the whole 2x2 matrix, so both decide alike.
    const bool two_way_push = c->cfg.pull == 0 && rb.R == 2 && ingress * 2 <= egress * 3 && egress * 2 <= ingress * 3;
    rb.pull = c->cfg.pull != 1 && !two_way_push;
    const uint64_t num = rb.R == 2 ? 31 : 6, den = rb.R == 2 ? 20 : 5;
    const bool grant = c->cfg.pull == 2 || (c->cfg.pull == 0 && !two_way_push && ingress * den <= egress * num);
    rb.send_post.assign(static_cast<size_t>(rb.R), Post{});
    const uint64_t ll_max = c->cfg.ll_max;
    for (int d = 0; d < rb.R; ++d) {
        const bool several = pair_is_multi(rb, rb.me, d);
        if (d == rb.me || rb.send_bytes[d] == 0 || (!several && ll_pair(plan, rb.me, d, rb.send_bytes[d], ll_max)))
            continue;
        Post p{};
        p.tag = 1;
        p.bytes = rb.send_bytes[d];
        p.mode = kSendPlain;
        const int w = several ? -1 : window_of(c, rb.send_ptr[d], rb.send_bytes[d]);
        if (w >= 0 && grant) {
            p.mode = kSendRegistered;
            p.win = static_cast<uint32_t>(w);
            p.off = rb.send_ptr[d] - c->windows[static_cast<size_t>(w)].base;
        }
        rb.send_post[static_cast<size_t>(d)] = p;
    }
    // a pair whose plan relays part of it takes pushes only: its relays push
    // into my port anyway, and pulling beside them was measured slower
    std::vector<char> relayed(static_cast<size_t>(rb.R), 0);
    for (const PairRoutes& pr : plan.pairs)
        if (pr.dst == rb.me)
            for (const Flow& f : pr.flows) relayed[static_cast<size_t>(pr.src)] |= pr.cands[static_cast<size_t>(f.cand)].via >= 0;
    rb.recv_post.assign(static_cast<size_t>(rb.R), Post{});
    for (int s = 0; s < rb.R; ++s) {
        const bool several = pair_is_multi(rb, s, rb.me);
        if (s == rb.me || rb.recv_bytes[s] == 0 || (!several && ll_pair(plan, s, rb.me, rb.recv_bytes[s], ll_max)))
            continue;
        Post p{};
        p.tag = 1;
        p.bytes = rb.recv_bytes[s];
        p.mode = kPostStaged;
        p.off = several ? 0 : rb.recv_ptr[s];  // several parts: the drain items carry absolute addresses
        if (several) {
            rb.recv_post[static_cast<size_t>(s)] = p;
            continue;
        }
        const int w = window_of(c, rb.recv_ptr[s], rb.recv_bytes[s]);
        if (w >= 0) {
            p.mode = kPostZeroCopy;
            p.win = static_cast<uint32_t>(w);
            p.off = rb.recv_ptr[s] - c->windows[static_cast<size_t>(w)].base;
        }
        const int dist = (rb.me - s + rb.R) % rb.R;  // NIMBLE_PUSH_DISTANCES: experiment, see push_distances()
        if (rb.pull && !relayed[static_cast<size_t>(s)] && !((push_distances() >> dist) & 1)) p.mode |= kPostPullRequest;
        rb.recv_post[static_cast<size_t>(s)] = p;
    }
}

constexpr size_t kCachedSchedules = 4;

// NIMBLE_PUSH_LANE=1: the push lane below (an experiment, off by default:
// measured 0.78 -> 0.56 of the bound at c3 r = 0.7, 64 MiB, W=4; see
// set_push_lane).
bool push_lane_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("NIMBLE_PUSH_LANE");
        return e && *e == '1';
    }();
    return on;
}

// The push lane: a port that declines pulls (it sends plain posts: its
// ingress dominates, profiles/r01_pull_policy.md) pushes its egress out while
// it pulls its ingress in.  Mixed in one queue, every CTA ends with peer
// stores in flight whose acknowledgements queue behind the saturated ingress,
// and its completion fence waits for them (2.6-12.9 us per CTA at 64 MiB,
// profiles/r02_trace_64_256mib_n4.txt).  With the pushes in their own queue,
// taken first by a share of the CTAs proportional to their bytes, the pushes
// finish early and the pulling CTAs end with a GPU-scope fence.  Direct
// pushes only (nvswitch model: no relay rings).
// Measured (profiles/r02_push_lane_*): the lane's CTAs push at ~5 GB/s each
// -- a port whose ingress is saturated gets its write acknowledgements late,
// and each SM has only so many stores in flight -- so 48 CTAs need 270 us for
// what all 148 CTAs, interleaving pushes with pulls, finish in 180 us.  Kept
// as an opt-in experiment.
void set_push_lane(Schedule& sc, const RankBuffers& rb) {
    uint64_t push = 0, other = 0;
    bool declined = false;
    for (const CutDesc& f : sc.cuts) {
        if (f.proto.kind == kPush) {
            push += f.bytes;
            declined |= rb.send_post[f.proto.peer].mode == kSendPlain;
        } else if (f.proto.kind == kPull) {
            other += f.bytes;
        } else if (f.proto.kind != kLocal && f.proto.kind != kForward) {
            return;  // relay hops: one queue (the original ordering argument)
        }
    }
    if (!declined || !push || !other) return;
    for (CutDesc& f : sc.cuts)
        if (f.proto.kind == kPush) {
            f.flags |= kCutPushLane;
            sc.n_push_lane += static_cast<uint32_t>(f.n);
        }
    sc.push_lane_bytes = push;
    sc.main_bytes = other;
}
void reap_retired(nimbleComm* c);

// Schedules whose flows fit the generator's parameter block are merged on
// the device (NIMBLE_HOST_SCHEDULE=1 forces the host merge + upload).
bool gen_on_device(const Schedule& sc) {
    static const bool host = [] {
        const char* e = std::getenv("NIMBLE_HOST_SCHEDULE");
        return e && *e == '1';
    }();
    return !host && sc.cuts.size() + sc.ll_cuts.size() <= static_cast<size_t>(kMaxGenCuts);
}

void fill_gen(GenArgs& g, const Schedule& sc, int R) {
    g.ncuts = static_cast<uint32_t>(sc.cuts.size() + sc.ll_cuts.size());
    g.nkeyed = static_cast<uint32_t>(sc.cuts.size());
    g.nitems = sc.nitems;
    g.nll = sc.n_ll_send + sc.n_ll_recv;
    g.R = static_cast<uint32_t>(R);
    g.n_push_lane = sc.n_push_lane;
    std::memset(g.post, 0, sizeof g.post);
    std::memset(g.send_post, 0, sizeof g.send_post);
    for (int r = 0; r < R && r < static_cast<int>(sc.posts.size()); ++r) g.post[r] = sc.posts[static_cast<size_t>(r)];
    for (int r = 0; r < R && r < static_cast<int>(sc.send_posts.size()); ++r)
        g.send_post[r] = sc.send_posts[static_cast<size_t>(r)];
    std::copy(sc.cuts.begin(), sc.cuts.end(), g.cuts);
    std::copy(sc.ll_cuts.begin(), sc.ll_cuts.end(), g.cuts + sc.cuts.size());
}

CachedSchedule& schedule_for(nimbleComm* c, uint64_t plan_id, const PlanResult& plan, const RankBuffers& rb,
                             cudaStream_t st) {
    std::vector<uint64_t> key = {plan_id, c->cfg.pipe_chunk, c->cfg.p2p_buffer,
                                 static_cast<uint64_t>(c->cfg.channels_per_peer), c->cfg.direct_chunk, c->cfg.push_chunk,
                                 c->cfg.ll_max};
    for (int r = 0; r < rb.R; ++r) {
        key.push_back(rb.send_ptr[r]);
        key.push_back(rb.send_bytes[r]);
        key.push_back(rb.recv_ptr[r]);
        key.push_back(rb.recv_bytes[r]);
        key.push_back(rb.recv_post[r].mode);
        key.push_back(rb.recv_post[r].win);
        key.push_back(rb.send_post[r].mode);
        key.push_back(rb.send_post[r].win);
    }
    for (const auto* parts : {&rb.send_parts, &rb.recv_parts}) {
        key.push_back(~0ull);  // list separator
        for (size_t p = 0; p < parts->size(); ++p)
            for (const auto& [ptr, bytes] : (*parts)[p]) {
                key.push_back(p);
                key.push_back(ptr);
                key.push_back(bytes);
            }
    }
    for (auto it = c->schedules.begin(); it != c->schedules.end(); ++it)
        if (it->key == key) {
            c->schedules.splice(c->schedules.begin(), c->schedules, it);
            return c->schedules.front();
        }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(st, &cap));
    if (cap != cudaStreamCaptureStatusNone)
        throw Error(nimbleInvalidUsage, "graph capture: run the same exchange once before capturing it "
                                        "(its schedule must be cached; capture does not allow uploads)");
    c->fast.cs = nullptr;  // entries may be recycled below
    const auto t0 = std::chrono::steady_clock::now();
    struct Timed {
        nimbleComm* c;
        std::chrono::steady_clock::time_point t0;
        ~Timed() {
            ++c->host.schedules;
            c->host.schedule_ns += static_cast<uint64_t>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
        }
    } timed{c, t0};
    reap_retired(c);
    CachedSchedule cs;
    cs.key = key;
    const uint64_t dchunk = c->cfg.direct_chunk ? c->cfg.direct_chunk : kDefaultDirectChunk;
    cs.sc = build_schedule(plan, rb, c->cfg.pipe_chunk, slot_count(c->cfg), dchunk,
                           c->cfg.push_chunk ? c->cfg.push_chunk : kDefaultPushChunk, c->cfg.ll_max);
    if (c->cfg.fabric == nimbleFabricNvSwitch && push_lane_enabled()) set_push_lane(cs.sc, rb);
    // Recycle the least recently used entry that no CUDA graph holds, once
    // kCachedSchedules of them exist: its buffers are rewritten on `st` after
    // its last launch (a stream wait on its event -- no host block, no
    // device-wide sync).
    size_t unpinned = 0;
    for (const CachedSchedule& e : c->schedules) unpinned += !e.pinned();
    if (unpinned >= kCachedSchedules) {
        for (auto it = std::prev(c->schedules.end());; --it) {
            if (!it->pinned()) {
                if (it->used) CUDA_TRY(cudaStreamWaitEvent(st, it->used, 0));
                cs.items = std::move(it->items);
                cs.posts = std::move(it->posts);
                cs.send_posts = std::move(it->send_posts);
                cs.finals = std::move(it->finals);
                cs.ll_items = std::move(it->ll_items);
                std::swap(cs.used, it->used);
                if (c->last_cs == &*it) c->last_cs = nullptr;
                c->schedules.erase(it);
                break;
            }
            if (it == c->schedules.begin()) break;
        }
    }
    if (!cs.used) CUDA_TRY(cudaEventCreateWithFlags(&cs.used, cudaEventDisableTiming));
    cs.finals.assign(cs.sc.final_waits, st, c->pool);
    if (gen_on_device(cs.sc)) {
        // the flows travel as kernel parameters; the device merges them
        cs.items.reserve(cs.sc.nitems, st, c->pool);
        cs.ll_items.reserve(cs.sc.n_ll_send + cs.sc.n_ll_recv, st, c->pool);
        cs.posts.reserve(static_cast<size_t>(rb.R), st, c->pool);
        cs.send_posts.reserve(static_cast<size_t>(rb.R), st, c->pool);
        GenArgs g;
        fill_gen(g, cs.sc, rb.R);
        g.items = cs.items.p;
        g.ll_items = cs.ll_items.p;
        g.posts = cs.posts.p;
        g.send_posts = cs.send_posts.p;
        CUDA_TRY(launch_gen(g, st));
    } else {
        materialize(cs.sc);
        cs.items.assign(cs.sc.items, st, c->pool);
        cs.posts.assign(cs.sc.posts, st, c->pool);
        cs.send_posts.assign(cs.sc.send_posts, st, c->pool);
        cs.ll_items.assign(cs.sc.ll_items, st, c->pool);
    }
    c->schedules.push_front(std::move(cs));
    return c->schedules.front();
}

// Drop every cached schedule (config change, deregistration, bench scope).
// Entries a CUDA graph still holds move to `retired` and stay allocated until
// the last such graph is destroyed; the rest are released once idle.
void drop_schedules(nimbleComm* c) {
    for (auto it = c->schedules.begin(); it != c->schedules.end();) {
        auto next = std::next(it);
        if (it->pinned()) c->retired.splice(c->retired.end(), c->schedules, it);
        else it->wait_idle();
        it = next;
    }
    c->schedules.clear();
    c->fast.cs = c->last_cs = nullptr;
}

// Free retired entries whose graphs are all gone.
void reap_retired(nimbleComm* c) {
    for (auto it = c->retired.begin(); it != c->retired.end();) {
        if (it->pinned()) {
            ++it;
        } else {
            it->wait_idle();
            it = c->retired.erase(it);
        }
    }
}

// A launch being captured into a CUDA graph keeps raw pointers to the
// entry's device buffers: pin the entry for the graph's lifetime (a user
// object retained by the graph decrements the pin count when the graph and
// all its executable instances are destroyed).
void pin_for_capture(CachedSchedule& cs, cudaStream_t st) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamGetCaptureInfo(st, &cap, nullptr, &graph, nullptr, nullptr));
    if (cap != cudaStreamCaptureStatusActive || !graph) return;
    auto* hold = new std::shared_ptr<GraphPins>(cs.pins);
    (*hold)->n.fetch_add(1);
    cudaUserObject_t obj = nullptr;
    cudaError_t e = cudaUserObjectCreate(
        &obj, hold,
        [](void* p) {
            auto* h = static_cast<std::shared_ptr<GraphPins>*>(p);
            (*h)->n.fetch_sub(1);
            delete h;
        },
        1, cudaUserObjectNoDestructorSync);
    if (e != cudaSuccess) {
        (*hold)->n.fetch_sub(1);
        delete hold;
        CUDA_TRY(e);
    }
    CUDA_TRY(cudaGraphRetainUserObject(graph, obj, 1, cudaGraphUserObjectMove));
}

// Programmatic dependent launch between consecutive exchanges (NIMBLE_PDL=0
// turns it off: A/B measurements, profilers that replay launches).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("NIMBLE_PDL");
        return !(e && *e == '0');
    }();
    return on;
}

// NIMBLE_CHAIN=0: every exchange waits for its predecessor's completion
// (griddepcontrol.wait) instead of chaining on its epoch (A/B measurements).
bool chain_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("NIMBLE_CHAIN");
        return !(e && *e == '0');
    }();
    return on;
}

// Pull stages in flight per CTA (NIMBLE_PULL_DEPTH=1..6 for experiments; 3).
uint32_t pull_depth() {
    static const uint32_t d = [] {
        const char* e = std::getenv("NIMBLE_PULL_DEPTH");
        const long v = e && *e ? std::strtol(e, nullptr, 10) : 3;
        return static_cast<uint32_t>(v < 1 ? 1 : (v > 6 ? 6 : v));
    }();
    return d;
}

// NIMBLE_TAIL_ITEMS=n: the last n items of the queue pull one stage at a
// time (experiment; 0 = off).
uint32_t tail_items() {
    static const uint32_t n = [] {
        const char* e = std::getenv("NIMBLE_TAIL_ITEMS");
        return static_cast<uint32_t>(e && *e ? std::strtoul(e, nullptr, 10) : 0);
    }();
    return n;
}

// NIMBLE_SPLIT_SIGNAL=0: the last CTA's warp 0 issues the completions owed to
// peers before its own waits (A/B; default: warp 1 issues them in parallel).
bool split_signal() {
    static const bool on = [] {
        const char* e = std::getenv("NIMBLE_SPLIT_SIGNAL");
        return !(e && *e == '0');
    }();
    return on;
}

bool launch_log() {
    static const bool on = [] {
        const char* e = std::getenv("NIMBLE_LAUNCH_LOG");
        return e && *e == '1';
    }();
    return on;
}

void launch(nimbleComm* c, CachedSchedule& cs, const RankBuffers& rb, cudaStream_t st) {
    LaunchArgs a{};
    a.items = cs.items.p;
    a.nitems = cs.sc.nitems;
    a.n_push_lane = cs.sc.n_push_lane;
    a.slots = slot_count(c->cfg);
    a.pipe_chunk = c->cfg.pipe_chunk;
    a.epoch = 0;  // the kernel takes it from c->view.epoch (device), see engine.cu
    a.comm = c->d_view;
    a.posts = cs.posts.p;
    a.send_posts = cs.send_posts.p;
    for (int r = 0; r < c->nranks; ++r) {
        a.send_bytes[r] = rb.send_bytes[r];
    }
    a.recv_direct = cs.sc.recv_direct;
    a.recv_zc = cs.sc.recv_zc;
    a.pull_req = cs.sc.pull_req;
    a.relay_writers = cs.sc.relay_writers;
    a.push_targets = cs.sc.push_targets;
    a.write_targets = cs.sc.write_targets;
    a.final_waits = cs.finals.p;
    a.nfinal = static_cast<uint32_t>(cs.sc.final_waits.size() / 2);
    a.n_ll_send = cs.sc.n_ll_send;
    a.n_ll_recv = cs.sc.n_ll_recv;
    a.ll_items = cs.ll_items.p;
    a.ll_senders = cs.sc.ll_senders;
    // Pulls keep at most 3 stages (96 KB) in flight per CTA: plenty for the
    // link, and a shorter drain (c3 at 4 GPUs, r = 0.5: 0.726 -> 0.773 of the
    // bound; other ratios within +-0.005; profiles/r01_pull_depth_n4.jsonl).
    a.pull_depth = pull_depth();
    a.tail_items = tail_items();
    a.split_signal = split_signal() ? 1u : 0u;
    a.local_only = 0;
    a.trace = c->d_trace;  // the kernel picks the timeline by epoch parity and resets the next one
    int ctas = c->cfg.ctas > 0 ? c->cfg.ctas : c->sms_share;
    // small exchanges: no more CTAs than items (each CTA costs a fence at exit)
    const size_t work = static_cast<size_t>(cs.sc.nitems) + cs.sc.n_ll_send + cs.sc.n_ll_recv;
    ctas = std::max(1, std::min({ctas, c->sms, static_cast<int>(std::max<size_t>(work, 1))}));
    if (cs.sc.n_push_lane) {  // CTAs for the push lane, by bytes (they join the main queue after)
        const double share = static_cast<double>(cs.sc.push_lane_bytes) /
                             static_cast<double>(cs.sc.push_lane_bytes + cs.sc.main_bytes);
        a.push_ctas = static_cast<uint32_t>(std::clamp(static_cast<int>(share * ctas + 0.5), 1, std::max(1, ctas - 1)));
    }
    // every rank launches even with nothing to move: its posts and done
    // flags are what its peers wait for.  Launches of one comm share its
    // scratch and flags, so a launch on another stream waits for the last one.
    // A launch on another stream than the previous one first waits for it
    // (same-stream launches are ordered already).  Not inside graph capture:
    // a captured launch is ordered by the graph the user builds.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(st, &cap));
    const bool eager = cap == cudaStreamCaptureStatusNone;
    if (eager && c->launched && st != c->last_stream) CUDA_TRY(cudaStreamWaitEvent(st, c->last_launch, 0));
    const bool pdl = c->colocated <= 1 && pdl_enabled();
    // chain on the previous exchange's epoch when it is this stream's
    // previous library launch (see engine.cu, exchange_kernel)
    const bool chain = eager && pdl && c->epoch_known && chain_enabled() && c->launched && st == c->chain_stream &&
                       c->chain_seq == g_launch_seq.load(std::memory_order_relaxed);
    a.prev_epoch = chain ? c->host_epoch : kEpochUnknown;
    CUDA_TRY(launch_exchange(a, ctas, st, pdl));
    if (eager) {
        ++c->host_epoch;
        c->chain_seq = g_launch_seq.load(std::memory_order_relaxed);
        c->chain_stream = st;
    } else {
        c->epoch_known = false;  // replays advance the device epoch unseen
    }
    if (launch_log()) {  // NIMBLE_LAUNCH_LOG=1: one stderr line per launch (debug aid)
        std::string sb, rbs;
        for (int r = 0; r < c->nranks; ++r) {
            sb += (r ? "," : "") + std::to_string(rb.send_bytes[r]);
            rbs += (r ? "," : "") + std::to_string(rb.recv_bytes[r]);
        }
        std::fprintf(stderr,
                     "[nimble] t %llu rank %d launch %llu ctas %d items %u ll_send %u ll_recv %u ll_senders %llx "
                     "pull_req %llx send [%s] recv [%s] stream %p%s\n",
                     static_cast<unsigned long long>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                                         std::chrono::system_clock::now().time_since_epoch())
                                                         .count() %
                                                     10000000000ll),
                     c->rank, static_cast<unsigned long long>(++c->host.launches), ctas, a.nitems, a.n_ll_send,
                     a.n_ll_recv, static_cast<unsigned long long>(a.ll_senders),
                     static_cast<unsigned long long>(a.pull_req), sb.c_str(), rbs.c_str(), static_cast<void*>(st),
                     eager ? "" : " (captured)");
    }
    if (eager) {
        CUDA_TRY(cudaEventRecord(c->last_launch, st));
        CUDA_TRY(cudaEventRecord(cs.used, st));
        c->last_stream = st;
        c->launched = true;
    } else {
        pin_for_capture(cs, st);
    }
}

void run_exchanges(std::vector<Exchange>& exs) {
    // single-process cliques: the members in this group must share the
    // data-path geometry (multi-process comms check it in SetConfig)
    for (Exchange& ex : exs)
        if (ex.comm->clique)
            for (Exchange& other : exs)
                if (other.comm->clique == ex.comm->clique &&
                    geometry_hash(other.comm->cfg) != geometry_hash(ex.comm->cfg))
                    throw Error(nimbleInvalidUsage, "group: comms of one clique disagree on the data-path geometry "
                                                    "(set the same config on every member)");
    // full demand matrix when the planner's model can route through relays
    std::map<nimbleComm*, std::vector<uint64_t>> full;
    for (Exchange& ex : exs) {
        nimbleComm* c = ex.comm;
        const int R = c->nranks;
        if (c->cfg.fabric != nimbleFabricAllToAll) continue;
        std::vector<uint64_t> m(static_cast<size_t>(R) * R, 0);
        if (c->boot) {  // host shared memory: the ranks share one machine (one NVLink box)
            std::vector<uint64_t> row(ex.rb.send_bytes);
            c->shm->allgather(row.data(), row.size() * sizeof(uint64_t), m.data(), c->view.timeout_ms);
        } else {
            for (Exchange& other : exs)
                if (other.comm->clique == c->clique)
                    for (int d = 0; d < R; ++d) m[static_cast<size_t>(other.comm->rank) * R + d] = other.rb.send_bytes[d];
            for (nimbleComm* peer : c->clique->comms) {
                bool present = false;
                for (Exchange& other : exs) present |= other.comm == peer;
                if (!present) throw Error(nimbleInvalidUsage, "group: every comm of the clique must take part");
            }
        }
        full[c] = std::move(m);
    }
    for (Exchange& ex : exs) {
        nimbleComm* c = ex.comm;
        DeviceGuard g(c->device);
        const int R = c->nranks, me = c->rank;
        std::vector<uint64_t> m;
        if (full.count(c)) {
            m = full[c];
        } else {  // nvswitch: one route per pair, my row and column decide my part
            m.assign(static_cast<size_t>(R) * R, 0);
            for (int p = 0; p < R; ++p) {
                if (p == me) continue;
                m[static_cast<size_t>(me) * R + p] = ex.rb.send_bytes[p];
                m[static_cast<size_t>(p) * R + me] = ex.rb.recv_bytes[p];
            }
        }
        for (int p = 0; p < R; ++p) m[static_cast<size_t>(p) * R + p] = 0;
        uint64_t plan_id = 0;
        std::shared_ptr<PlanResult> plan = plan_for(c, m, &plan_id);
        fill_posts(c, ex.rb, *plan);
        CachedSchedule& cs = schedule_for(c, plan_id, *plan, ex.rb, ex.stream);
        std::vector<cudaEvent_t> evs;
        for (cudaStream_t o : ex.others) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CUDA_TRY(cudaEventRecord(e, o));
            CUDA_TRY(cudaStreamWaitEvent(ex.stream, e, 0));
            evs.push_back(e);
        }
        launch(c, cs, ex.rb, ex.stream);
        c->last_cs = &cs;
        c->last_rb = ex.rb;
        for (size_t i = 0; i < ex.others.size(); ++i) {
            CUDA_TRY(cudaEventRecord(evs[i], ex.stream));
            CUDA_TRY(cudaStreamWaitEvent(ex.others[i], evs[i], 0));
            cudaEventDestroy(evs[i]);
        }
    }
}

void flush_group() {
    std::vector<PendingOp> ops;
    ops.swap(g_pending);
    std::vector<nimbleComm*> order;
    std::map<nimbleComm*, std::vector<PendingOp*>> by_comm;
    for (PendingOp& op : ops) {
        if (!by_comm.count(op.comm)) order.push_back(op.comm);
        by_comm[op.comm].push_back(&op);
    }
    std::vector<Exchange> exs;
    for (nimbleComm* c : order) exs.push_back(make_exchange(c, by_comm[c]));
    run_exchanges(exs);
}

nimbleResult_t enqueue(PendingOp&& op) {
    return guarded([&] {
        if (!op.comm) throw Error(nimbleInvalidArgument, "null comm");
        g_pending.push_back(std::move(op));
        if (g_group_depth == 0) flush_group();
    });
}

// ---------------------------------------------------------------- registration

void* register_window(nimbleComm* c, void* buff, size_t size) {
    DeviceGuard g(c->device);
    uint32_t id = static_cast<uint32_t>(c->windows.size());
    if (id >= kMaxWindows) throw Error(nimbleInvalidUsage, "register: too many windows");
    Window w;
    w.live = buff != nullptr && size > 0;
    w.base = reinterpret_cast<uint64_t>(buff);
    w.size = size;
    if (c->boot) {
        struct Blob {
            cudaIpcMemHandle_t h;
            uint64_t offset, size, addr;
            int32_t live, pid;
        } mine{};
        if (w.live) {
            auto [base, asz] = allocation_of(buff);
            (void)asz;
            CUDA_TRY(cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)));
            mine.offset = w.base - base;
        }
        mine.size = size;
        mine.live = w.live;
        mine.addr = w.base;
        mine.pid = ::getpid();
        std::vector<Blob> all(static_cast<size_t>(c->nranks));
        c->boot->allgather(&mine, sizeof mine, all.data());
        for (int r = 0; r < c->nranks; ++r) {
            const Blob& b = all[static_cast<size_t>(r)];
            uint64_t addr = 0;
            if (r == c->rank) {
                addr = w.base;
            } else if (b.live && b.pid == mine.pid) {
                addr = b.addr;  // a rank of this process: its pointer as it is
            } else if (b.live) {
                void* p = ipc_cache().acquire(b.h);
                w.opened.push_back(p);
                addr = reinterpret_cast<uint64_t>(p) + b.offset;
            }
            c->win_table[static_cast<size_t>(id) * kMaxRanks + r] = addr;
        }
        h2d(c, c->d_win_table + static_cast<size_t>(id) * kMaxRanks, &c->win_table[static_cast<size_t>(id) * kMaxRanks],
            sizeof(uint64_t) * kMaxRanks);
    } else {
        // single process: peers see each other's pointers directly; window k of
        // every comm in the clique is published as soon as it is registered
        for (nimbleComm* peer : c->clique->comms) {
            peer->win_table[static_cast<size_t>(id) * kMaxRanks + c->rank] = w.base;
            DeviceGuard pg(peer->device);
            h2d(peer, peer->d_win_table + static_cast<size_t>(id) * kMaxRanks + c->rank, &w.base, sizeof(uint64_t));
        }
    }
    c->windows.push_back(std::move(w));
    c->fast.cs = nullptr;  // new window: posts of the same buffers may change
    c->view.nwin = static_cast<uint32_t>(c->windows.size());
    return reinterpret_cast<void*>(static_cast<uintptr_t>(id) + 1);
}

// ---------------------------------------------------------------- bench

double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v.empty() ? 0.0 : v[v.size() / 2];
}

void bench_matrix(nimbleComm* c, const std::vector<uint64_t>& m, int warmup, int iters, nimbleBenchResult* out) {
    if (!c->boot) throw Error(nimbleInvalidUsage, "bench entry points need one process per GPU (nimbleCommInitRank)");
    if (!out) throw Error(nimbleInvalidArgument, "bench: null result");
    DeviceGuard g(c->device);
    const int R = c->nranks, me = c->rank;
    std::vector<size_t> sc(R), sd(R), rc(R), rd(R);
    size_t stot = 0, rtot = 0;
    for (int p = 0; p < R; ++p) {
        sc[p] = m[static_cast<size_t>(me) * R + p];
        sd[p] = stot;
        stot += sc[p];
        rc[p] = m[static_cast<size_t>(p) * R + me];
        rd[p] = rtot;
        rtot += rc[p];
    }
    // Buffers and windows are released on every exit path (the windows' IPC
    // mappings are dropped locally; the comm's peers do the same on theirs).
    struct Scope {
        nimbleComm* c;
        std::vector<void*> bufs;
        size_t first_window;
        ~Scope() {
            if (c->bench_stream) cudaStreamSynchronize(c->bench_stream);
            for (size_t k = first_window; k < c->windows.size(); ++k) {
                c->windows[k].live = false;
                for (void* p : c->windows[k].opened) ipc_cache().release(p);
                c->windows[k].opened.clear();
            }
            drop_schedules(c);
            for (void* b : bufs) cudaFree(b);
        }
    } scope{c, {}, c->windows.size()};
    auto alloc = [&scope](size_t n) {
        void* p = nullptr;
        CUDA_TRY(cudaMalloc(&p, n));
        scope.bufs.push_back(p);
        return p;
    };
    auto* sbuf = static_cast<uint8_t*>(alloc(std::max<size_t>(stot, 16)));
    auto* rbuf = static_cast<uint8_t*>(alloc(std::max<size_t>(rtot, 16)));
    auto* bad = static_cast<uint64_t*>(alloc(sizeof(uint64_t)));
    const uint64_t seed = 1;
    if (!c->bench_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->bench_stream, cudaStreamNonBlocking));
    cudaStream_t st = c->bench_stream;
    for (int p = 0; p < R; ++p) CUDA_TRY(launch_fill(sbuf + sd[p], 0, sc[p], seed, me, p, st));
    register_window(c, rbuf, std::max<size_t>(rtot, 16));
    register_window(c, sbuf, std::max<size_t>(stot, 16));  // ingress-heavy receivers may pull
    auto once = [&] {
        nimbleResult_t r = nimbleAlltoAllv(sbuf, sc.data(), sd.data(), rbuf, rc.data(), rd.data(), nimbleUint8, c, st);
        if (r != nimbleSuccess) throw Error(r, g_last_error);
    };
    for (int i = 0; i < warmup; ++i) once();
    CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(iters));
    for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
    std::vector<double> mine(static_cast<size_t>(iters));
    for (int i = 0; i < iters; ++i) {
        c->boot->barrier();
        CUDA_TRY(cudaEventRecord(ev[2 * i], st));
        once();
        CUDA_TRY(cudaEventRecord(ev[2 * i + 1], st));
        CUDA_TRY(cudaStreamSynchronize(st));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        mine[static_cast<size_t>(i)] = ms * 1e-3;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    std::vector<double> all(mine.size() * static_cast<size_t>(R));
    c->boot->allgather(mine.data(), mine.size() * sizeof(double), all.data());
    std::vector<double> worst(mine.size(), 0.0);
    for (int r = 0; r < R; ++r)
        for (size_t i = 0; i < mine.size(); ++i) worst[i] = std::max(worst[i], all[static_cast<size_t>(r) * mine.size() + i]);
    // verification pass on a cleared buffer
    CUDA_TRY(cudaMemsetAsync(rbuf, 0, std::max<size_t>(rtot, 16), st));
    c->boot->barrier();
    once();
    CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(uint64_t), st));
    for (int p = 0; p < R; ++p) CUDA_TRY(launch_check(rbuf + rd[p], 0, rc[p], seed, p, me, bad, st));
    uint64_t my_bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&my_bad, bad, sizeof my_bad, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (c->h_status[0]) throw Error(nimbleRemoteError, "bench: forwarding engine reported async error " +
                                                           std::to_string(c->h_status[0]));
    std::vector<uint64_t> bads(static_cast<size_t>(R));
    c->boot->allgather(&my_bad, sizeof my_bad, bads.data());
    uint64_t total = 0, worst_port = 0;
    for (int v = 0; v < R; ++v) {
        uint64_t eg = 0, ig = 0;
        for (int p = 0; p < R; ++p) {
            eg += v == p ? 0 : m[static_cast<size_t>(v) * R + p];
            ig += v == p ? 0 : m[static_cast<size_t>(p) * R + v];
            total += m[static_cast<size_t>(v) * R + p];
        }
        worst_port = std::max({worst_port, eg, ig});
    }
    std::memset(out, 0, sizeof *out);
    out->seconds_median = median(worst);
    out->seconds_min = worst.empty() ? 0.0 : *std::min_element(worst.begin(), worst.end());
    out->total_bytes = total;
    out->gbps_effective = out->seconds_median > 0 ? static_cast<double>(total) / out->seconds_median / 1e9 : 0.0;
    out->bound_seconds = static_cast<double>(worst_port) / c->cfg.nvlink_bytes_per_s;
    for (uint64_t b : bads) out->mismatches += b;
    {
        std::vector<uint64_t> mm(m);
        for (int p = 0; p < R; ++p) mm[static_cast<size_t>(p) * R + p] = 0;
        const LinkModel lm = comm_model(c);
        Demand d;
        d.ranks = R;
        d.bytes = mm;
        PlanResult pr = mcf_plan(lm, R, lm.gpus, d, to_params(&c->cfg.planner));
        out->plan_seconds = pr.stats.wall_seconds;
        for (const PairRoutes& p : pr.pairs)
            for (const Flow& f : p.flows) out->relay_flows += p.cands[static_cast<size_t>(f.cand)].via >= 0;
    }
    c->boot->barrier();  // no peer touches these windows any more
}

}  // namespace
}  // namespace nb

using nb::fail;
using nb::guarded;

extern "C" {

nimbleResult_t nimbleCommConfigDefault(nimbleCommConfig* cfg) {
    if (!cfg) return fail(nimbleInvalidArgument, "config: null");
    nb::default_config(cfg, 0);
    return nimbleSuccess;
}

nimbleResult_t nimbleGetUniqueId(nimbleUniqueId* id) {
    return guarded([&] {
        if (!id) throw nb::Error(nimbleInvalidArgument, "null unique id");
        nb::bootstrap_root(id);
    });
}

nimbleResult_t nimbleCommInitRank(nimbleComm_t* out, int nranks, nimbleUniqueId id, int rank) {
    return guarded([&] {
        if (!out) throw nb::Error(nimbleInvalidArgument, "null comm");
        if (nranks < 1 || nranks > nb::kMaxRanks || rank < 0 || rank >= nranks)
            throw nb::Error(nimbleInvalidArgument, "comm: bad rank / size (max 32 ranks)");
        auto c = std::make_unique<nimbleComm>();
        c->rank = rank;
        c->nranks = nranks;
        CUDA_TRY(cudaGetDevice(&c->device));
        nb::default_config(&c->cfg, nranks);
        c->boot = nb::bootstrap_connect(id, rank, nranks);
        c->shm = std::make_unique<nb::ShmAllgather>(id, *c->boot);
        nb::setup_common(c.get());
        nb::setup_regions(c.get(), false);
        nb::upload_view(c.get());
        c->boot->barrier();
        *out = c.release();
    });
}

nimbleResult_t nimbleCommInitAll(nimbleComm_t* comms, int ndev, const int* devlist) {
    return guarded([&] {
        if (!comms || ndev < 1 || ndev > nb::kMaxRanks) throw nb::Error(nimbleInvalidArgument, "comm: bad device list");
        auto clique = std::make_shared<nb::Clique>();
        std::vector<std::unique_ptr<nimbleComm>> made;
        for (int r = 0; r < ndev; ++r) {
            auto c = std::make_unique<nimbleComm>();
            c->rank = r;
            c->nranks = ndev;
            c->device = devlist ? devlist[r] : r;
            c->clique = clique;
            nb::default_config(&c->cfg, ndev);
            nb::setup_common(c.get());
            nb::setup_regions(c.get(), true);
            clique->comms.push_back(c.get());
            made.push_back(std::move(c));
        }
        for (auto& c : made) {
            nb::DeviceGuard g(c->device);
            c->colocated = 0;
            for (auto& p : made) {
                c->peer_ctrl[static_cast<size_t>(p->rank)] = p->ctrl;
                c->peer_staging[static_cast<size_t>(p->rank)] = p->staging;
                if (p->device != c->device) nb::enable_peer(p->device);
                else ++c->colocated;  // a repeated device: co-resident ranks
            }
            nb::set_share(c.get());
            nb::upload_view(c.get());
        }
        for (int r = 0; r < ndev; ++r) comms[r] = made[static_cast<size_t>(r)].release();
    });
}

nimbleComm::~nimbleComm() {
    // never throws: a comm whose init failed may have no usable device
    int prev = -1;
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        prev = -1;
    }
    for (nb::Window& w : windows)
        for (void* p : w.opened) nb::ipc_cache().release(p);
    windows.clear();
    for (auto& e : schedules) e.wait_idle();
    for (auto& e : retired) e.wait_idle();
    schedules.clear();
    retired.clear();
    fast.cs = last_cs = nullptr;
    if (clique) {
        // Peers' engine grids of this clique write into my ctrl region at
        // their epilogue (done / pulled / LL acks) whether or not they
        // exchanged data with me: the regions outlive me until the last
        // member of the clique is gone (~Clique syncs every device first).
        clique->deferred.push_back({device, ctrl, staging});
        ctrl = staging = nullptr;
    }
    nb::free_regions(this);
    cudaFree(d_view);
    cudaFree(d_win_table);
    cudaFree(d_scratch);
    cudaFree(d_epoch);
    if (d_trace) cudaFree(d_trace);
    if (d_stats) cudaFree(d_stats);
    if (h_status) cudaFreeHost(h_status);
    if (bench_stream) cudaStreamDestroy(bench_stream);  // created by the first bench entry point call
    if (pool) cudaMemPoolDestroy(pool);  // released once its frees complete
    if (last_launch) cudaEventDestroy(last_launch);
    cudaGetLastError();
    if (prev >= 0) cudaSetDevice(prev);
}

nimbleResult_t nimbleCommDestroy(nimbleComm_t c) {
    if (!c) return nimbleSuccess;
    return guarded([&] {
        {
            nb::DeviceGuard g(c->device);
            nb::quiesce(c);
            if (c->boot) c->boot->barrier();  // nobody touches my regions any more
        }
        if (c->clique) {
            auto& v = c->clique->comms;
            v.erase(std::remove(v.begin(), v.end(), c), v.end());
        }
        delete c;  // ~nimbleComm frees everything
    });
}

nimbleResult_t nimbleCommCount(const nimbleComm_t c, int* n) {
    if (!c || !n) return fail(nimbleInvalidArgument, "null argument");
    *n = c->nranks;
    return nimbleSuccess;
}

nimbleResult_t nimbleCommUserRank(const nimbleComm_t c, int* r) {
    if (!c || !r) return fail(nimbleInvalidArgument, "null argument");
    *r = c->rank;
    return nimbleSuccess;
}

nimbleResult_t nimbleCommCuDevice(const nimbleComm_t c, int* d) {
    if (!c || !d) return fail(nimbleInvalidArgument, "null argument");
    *d = c->device;
    return nimbleSuccess;
}

nimbleResult_t nimbleCommGetAsyncError(nimbleComm_t c, nimbleResult_t* err) {
    if (!c || !err) return fail(nimbleInvalidArgument, "null argument");
    const uint32_t code = *reinterpret_cast<volatile uint32_t*>(c->h_status);
    *err = code == 0 ? nimbleSuccess : (code == 5 || code == 6) ? nimbleInvalidUsage : nimbleRemoteError;
    if (code) {
        static const char* what[] = {"", "timeout waiting for a receiver's post", "timeout waiting for a staging slot",
                                     "timeout waiting for a relayed chunk", "timeout waiting for a writer's done flag",
                                     "send and receive counts disagree across ranks",
                                     "relay routes need a registered receive buffer",
                                     "timeout waiting for a relay to drain",
                                     "a post was overwritten before it was read (protocol violation)",
                                     "timeout on a low-latency (LL) slot",
                                     "a work item fell outside its segment or staging slot (scheduler bug; nothing "
                                     "was written)"};
        nb::g_last_error = code < sizeof what / sizeof what[0] ? what[code] : "unknown device error";
        // where: peer (0xff = unknown; bit 7 = the other direction: a pull, or
        // an LL receive) and the epoch's low 16 bits
        const uint32_t detail = reinterpret_cast<volatile uint32_t*>(c->h_status)[1];
        const uint32_t peer = detail >> 16 & 0xff;
        nb::g_last_error += " (rank " + std::to_string(c->rank) + ", peer " +
                            (peer == 0xff ? std::string("?") : std::to_string(peer & 0x7f) +
                                                                   ((peer & 0x80) ? " [in]" : "")) +
                            ", epoch " + std::to_string(detail & 0xffff) + ")";
        if (code == 9) {  // LL: what the polled line held
            volatile uint32_t* st = reinterpret_cast<volatile uint32_t*>(c->h_status);
            nb::g_last_error += " [line " + std::to_string(st[4]) + " of piece " + std::to_string(st[5]) +
                                " held flags " + std::to_string(st[2]) + "/" + std::to_string(st[3]) + "]";
        }
    }
    return nimbleSuccess;
}

nimbleResult_t nimbleCommSetConfig(nimbleComm_t c, const nimbleCommConfig* cfg) {
    return guarded([&] {
        if (!c || !cfg) throw nb::Error(nimbleInvalidArgument, "null argument");
        nimbleCommConfig next = *cfg;
        if (next.gpus_per_node <= 0) next.gpus_per_node = c->nranks;
        if (next.fabric == nimbleFabricAllToAll && next.gpus_per_node != c->nranks)
            throw nb::Error(nimbleInvalidArgument, "config: the mesh model must have one GPU per rank");
        if (!(next.nvlink_bytes_per_s > 0)) throw nb::Error(nimbleInvalidArgument, "config: bandwidth must be positive");
        nb::slot_count(next);
        nb::to_params(&next.planner);
        if (next.ll_max > nb::kLLMaxData)
            throw nb::Error(nimbleInvalidArgument, "config: ll_max above the LL slot size (1 MiB)");
        const bool regrow = next.pipe_chunk != c->cfg.pipe_chunk || next.p2p_buffer != c->cfg.p2p_buffer ||
                            next.channels_per_peer != c->cfg.channels_per_peer ||
                            nb::ring_count(c, next) != nb::ring_count(c, c->cfg);
        nb::DeviceGuard g(c->device);
        if (c->boot) {  // collective: every rank must bring the same data-path geometry
            const uint64_t mine = nb::geometry_hash(next);
            std::vector<uint64_t> all(static_cast<size_t>(c->nranks));
            c->boot->allgather(&mine, sizeof mine, all.data());
            for (uint64_t h : all)
                if (h != mine)
                    throw nb::Error(nimbleInvalidUsage, "config: ranks disagree on the data-path geometry "
                                                        "(chunk sizes, staging, LL limit, fabric model)");
        }
        if (regrow && c->clique) {
            // one process: swap my staging region under every member's view
            // (they are idle between grouped calls; wait for their last launches)
            for (nimbleComm* p : c->clique->comms) {
                nb::DeviceGuard pg(p->device);
                nb::quiesce(p);
            }
            c->cfg = next;
            CUDA_TRY(cudaFree(c->staging));
            c->staging = nullptr;
            c->staging_bytes = nb::staging_size(c);
            CUDA_TRY(cudaMalloc(&c->staging, std::max<uint64_t>(c->staging_bytes, 256)));
            for (nimbleComm* p : c->clique->comms) {
                p->peer_staging[static_cast<size_t>(c->rank)] = c->staging;
                nb::DeviceGuard pg(p->device);
                nb::upload_view(p);
            }
        } else if (regrow) {
            nb::quiesce(c);
            if (c->boot) c->boot->barrier();
            nb::free_regions(c);  // nulls the pointers: a failing setup below leaves nothing to double-free
            c->cfg = next;
            nb::setup_regions(c, false);
            nb::zero(c, c->d_epoch, sizeof(uint64_t));  // fresh flags: epochs restart
            c->host_epoch = 0;
            nb::upload_view(c);
        }
        c->cfg = next;
        nb::upload_view(c);
        c->plans.clear();
        nb::drop_schedules(c);
        if (c->boot) c->boot->barrier();
    });
}

nimbleResult_t nimbleCommGetConfig(nimbleComm_t c, nimbleCommConfig* cfg) {
    if (!c || !cfg) return fail(nimbleInvalidArgument, "null argument");
    *cfg = c->cfg;
    return nimbleSuccess;
}

nimbleResult_t nimbleCommRegister(const nimbleComm_t c, void* buff, size_t size, void** handle) {
    return guarded([&] {
        if (!c || !handle) throw nb::Error(nimbleInvalidArgument, "null argument");
        *handle = nb::register_window(c, buff, size);
        nb::upload_view(c);
    });
}

nimbleResult_t nimbleCommDeregister(const nimbleComm_t c, void* handle) {
    return guarded([&] {
        if (!c) throw nb::Error(nimbleInvalidArgument, "null comm");
        const size_t id = reinterpret_cast<uintptr_t>(handle) - 1;
        if (id >= c->windows.size() || !c->windows[id].live) throw nb::Error(nimbleInvalidArgument, "bad handle");
        nb::DeviceGuard g(c->device);
        nb::quiesce(c);
        if (c->boot) c->boot->barrier();
        for (void* p : c->windows[id].opened) nb::ipc_cache().release(p);
        c->windows[id].opened.clear();
        c->windows[id].live = false;
        nb::drop_schedules(c);
    });
}

nimbleResult_t nimbleMemAlloc(void** ptr, size_t size) {
    return guarded([&] {
        if (!ptr) throw nb::Error(nimbleInvalidArgument, "null pointer");
        CUDA_TRY(cudaMalloc(ptr, std::max<size_t>(size, 16)));
    });
}

nimbleResult_t nimbleMemFree(void* ptr) {
    return guarded([&] { CUDA_TRY(cudaFree(ptr)); });
}

nimbleResult_t nimbleGroupStart(void) {
    ++nb::g_group_depth;
    return nimbleSuccess;
}

nimbleResult_t nimbleGroupEnd(void) {
    if (nb::g_group_depth <= 0) return fail(nimbleInvalidUsage, "group end without start");
    if (--nb::g_group_depth > 0) return nimbleSuccess;
    return guarded([&] { nb::flush_group(); });
}

nimbleResult_t nimbleSend(const void* sendbuff, size_t count, nimbleDataType_t dt, int peer, nimbleComm_t comm,
                          void* stream) {
    return guarded([&] {
        if (!comm || peer < 0 || peer >= comm->nranks) throw nb::Error(nimbleInvalidArgument, "send: bad peer");
        nb::PendingOp op{nb::PendingOp::Send, comm, static_cast<cudaStream_t>(stream), peer,
                         reinterpret_cast<uint64_t>(sendbuff), count * nb::elem_size(dt), 0, 0, {}, {}, {}, {}};
        nimbleResult_t r = nb::enqueue(std::move(op));
        if (r != nimbleSuccess) throw nb::Error(r, nb::g_last_error);
    });
}

nimbleResult_t nimbleRecv(void* recvbuff, size_t count, nimbleDataType_t dt, int peer, nimbleComm_t comm, void* stream) {
    return guarded([&] {
        if (!comm || peer < 0 || peer >= comm->nranks) throw nb::Error(nimbleInvalidArgument, "recv: bad peer");
        nb::PendingOp op{nb::PendingOp::Recv, comm, static_cast<cudaStream_t>(stream), peer,
                         reinterpret_cast<uint64_t>(recvbuff), count * nb::elem_size(dt), 0, 0, {}, {}, {}, {}};
        nimbleResult_t r = nb::enqueue(std::move(op));
        if (r != nimbleSuccess) throw nb::Error(r, nb::g_last_error);
    });
}

nimbleResult_t nimbleAlltoAllv(const void* sendbuff, const size_t sendcounts[], const size_t sdispls[], void* recvbuff,
                               const size_t recvcounts[], const size_t rdispls[], nimbleDataType_t dt,
                               nimbleComm_t comm, void* stream) {
    const auto t0 = std::chrono::steady_clock::now();
    struct Timed {
        nimbleComm* c;
        std::chrono::steady_clock::time_point t0;
        ~Timed() {
            if (!c) return;
            const uint64_t ns = static_cast<uint64_t>(
                std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
            ++c->host.calls;
            c->host.ns += ns;
            c->host.ns_max = std::max(c->host.ns_max, ns);
        }
    } timed{comm, t0};
    return guarded([&] {
        if (!comm || !sendcounts || !sdispls || !recvcounts || !rdispls)
            throw nb::Error(nimbleInvalidArgument, "alltoallv: null argument");
        const size_t es = nb::elem_size(dt);
        const int R = comm->nranks;
        // The same stand-alone call as last time (same buffers and counts, no
        // group, nvswitch model: the plan needs only this rank's row and
        // column) relaunches its cached schedule directly.
        uint64_t key[2 + 4 * nb::kMaxRanks];
        key[0] = reinterpret_cast<uint64_t>(sendbuff);
        key[1] = reinterpret_cast<uint64_t>(recvbuff);
        for (int p = 0; p < R; ++p) {
            key[2 + 4 * p] = sendcounts[p] * es;
            key[3 + 4 * p] = sdispls[p] * es;
            key[4 + 4 * p] = recvcounts[p] * es;
            key[5 + 4 * p] = rdispls[p] * es;
        }
        const size_t key_bytes = sizeof(uint64_t) * (2 + 4 * static_cast<size_t>(R));
        const bool standalone = nb::g_group_depth == 0 && comm->cfg.fabric == nimbleFabricNvSwitch;
        if (standalone && comm->fast.cs && std::memcmp(key, comm->fast.key, key_bytes) == 0) {
            nb::DeviceGuard g(comm->device);
            nb::launch(comm, *comm->fast.cs, comm->fast.rb, static_cast<cudaStream_t>(stream));
            return;
        }
        nb::PendingOp op{nb::PendingOp::AllToAllV, comm, static_cast<cudaStream_t>(stream), -1, 0, 0,
                         reinterpret_cast<uint64_t>(sendbuff), reinterpret_cast<uint64_t>(recvbuff), {}, {}, {}, {}};
        for (int p = 0; p < R; ++p) {
            op.sbytes.push_back(key[2 + 4 * p]);
            op.soff.push_back(key[3 + 4 * p]);
            op.rbytes.push_back(key[4 + 4 * p]);
            op.roff.push_back(key[5 + 4 * p]);
        }
        nimbleResult_t r = nb::enqueue(std::move(op));
        if (r != nimbleSuccess) throw nb::Error(r, nb::g_last_error);
        if (standalone && comm->last_cs) {
            std::memcpy(comm->fast.key, key, key_bytes);
            comm->fast.cs = comm->last_cs;
            comm->fast.rb = comm->last_rb;
        }
    });
}

nimbleResult_t nimbleAlltoAll(const void* sendbuff, void* recvbuff, size_t count, nimbleDataType_t dt,
                              nimbleComm_t comm, void* stream) {
    if (!comm) return fail(nimbleInvalidArgument, "alltoall: null comm");
    std::vector<size_t> counts(static_cast<size_t>(comm->nranks), count), displs(static_cast<size_t>(comm->nranks));
    for (int p = 0; p < comm->nranks; ++p) displs[static_cast<size_t>(p)] = count * static_cast<size_t>(p);
    return nimbleAlltoAllv(sendbuff, counts.data(), displs.data(), recvbuff, counts.data(), displs.data(), dt, comm,
                           stream);
}

nimbleResult_t nimbleFillPayload(void* buf, uint64_t first, uint64_t n, uint64_t seed, int s, int d, void* stream) {
    return guarded([&] { CUDA_TRY(nb::launch_fill(buf, first, n, seed, s, d, static_cast<cudaStream_t>(stream))); });
}

nimbleResult_t nimbleCheckPayload(const void* buf, uint64_t first, uint64_t n, uint64_t seed, int s, int d,
                                  uint64_t* bad, void* stream) {
    return guarded([&] {
        CUDA_TRY(nb::launch_check(buf, first, n, seed, s, d, bad, static_cast<cudaStream_t>(stream)));
    });
}

nimbleResult_t nimbleBenchMatrix(nimbleComm_t c, const uint64_t* matrix, int warmup, int iters,
                                 nimbleBenchResult* out) {
    return guarded([&] {
        if (!c || !matrix || iters < 1 || warmup < 0) throw nb::Error(nimbleInvalidArgument, "bench: bad argument");
        std::vector<uint64_t> m(matrix, matrix + static_cast<size_t>(c->nranks) * c->nranks);
        nb::bench_matrix(c, m, warmup, iters, out);
    });
}

nimbleResult_t nimbleBenchP2P(nimbleComm_t c, uint64_t bytes, int src, int dst, int warmup, int iters,
                              nimbleBenchResult* out) {
    return guarded([&] {
        if (!c) throw nb::Error(nimbleInvalidArgument, "bench: null comm");
        nb::Demand d = nb::demand_p2p(c->nranks, src, dst, bytes);
        nb::bench_matrix(c, d.bytes, warmup, iters, out);
    });
}

nimbleResult_t nimbleBenchSkewed(nimbleComm_t c, uint64_t per_rank, double ratio, int hot, int warmup, int iters,
                                 nimbleBenchResult* out) {
    return guarded([&] {
        if (!c) throw nb::Error(nimbleInvalidArgument, "bench: null comm");
        nb::Demand d = nb::demand_skewed(c->nranks, per_rank, ratio, hot, false);
        nb::bench_matrix(c, d.bytes, warmup, iters, out);
    });
}

nimbleResult_t nimbleCommDebugTrace(nimbleComm_t c, uint64_t* out, int n) {
    return guarded([&] {
        if (!c || !out || n < nb::kTraceSlots) throw nb::Error(nimbleInvalidArgument, "trace: bad argument");
        if (!c->d_trace) throw nb::Error(nimbleInvalidUsage, "trace: set NIMBLE_TRACE=1 before creating the comm");
        nb::DeviceGuard g(c->device);
        nb::quiesce(c);
        uint64_t epoch = 0;  // the latest launch's timeline: buffer epoch & 1
        CUDA_TRY(cudaMemcpy(&epoch, c->d_epoch, sizeof epoch, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(out, c->d_trace + (epoch & 1) * nb::kTraceWords,
                            sizeof(uint64_t) * static_cast<size_t>(std::min(n, nb::kTraceWords)), cudaMemcpyDeviceToHost));
    });
}

nimbleResult_t nimbleCommGetStats(nimbleComm_t c, nimbleCommStats* out, int reset) {
    return guarded([&] {
        if (!c || !out) throw nb::Error(nimbleInvalidArgument, "stats: null argument");
        if (!c->d_stats) throw nb::Error(nimbleInvalidUsage, "stats: set NIMBLE_STATS=1 before creating the comm");
        static_assert(sizeof(nimbleCommStats) == sizeof(nb::DeviceStats), "stats layout");
        nb::DeviceGuard g(c->device);
        nb::quiesce(c);
        CUDA_TRY(cudaMemcpy(out, c->d_stats, sizeof *out, cudaMemcpyDeviceToHost));
        out->host_calls = c->host.calls;
        out->host_ns = c->host.ns;
        out->host_ns_max = c->host.ns_max;
        out->plans_built = c->host.plans;
        out->plan_ns = c->host.plan_ns;
        out->schedules_built = c->host.schedules;
        out->schedule_ns = c->host.schedule_ns;
        out->host_pad = 0;
        if (reset) {
            nb::zero(c, c->d_stats, sizeof(nb::DeviceStats));
            c->host = {};
        }
    });
}

nimbleResult_t nimbleBootstrapShmAllgather(const nimbleUniqueId* id, int rank, int nranks, const void* in, size_t n,
                                           void* out, int rounds) {
    return guarded([&] {
        if (!id || rounds < 1 || n + 8 > nb::ShmAllgather::kRecord || (n && (!in || !out)))
            throw nb::Error(nimbleInvalidArgument, "bootstrap: bad argument");
        auto b = nb::bootstrap_connect(*id, rank, nranks);
        nb::ShmAllgather shm(*id, *b);
        std::vector<uint8_t> rec(n + 8), all((n + 8) * static_cast<size_t>(nranks));
        for (int k = 1; k <= rounds; ++k) {
            const uint64_t tag = static_cast<uint64_t>(k) << 8 | static_cast<uint64_t>(rank);
            std::memcpy(rec.data(), &tag, 8);
            if (n) std::memcpy(rec.data() + 8, in, n);
            shm.allgather(rec.data(), rec.size(), all.data(), 60000);
            for (int r = 0; r < nranks; ++r) {  // every record is this round's, from its rank
                uint64_t t = 0;
                std::memcpy(&t, all.data() + static_cast<size_t>(r) * rec.size(), 8);
                if (t != (static_cast<uint64_t>(k) << 8 | static_cast<uint64_t>(r)))
                    throw nb::Error(nimbleInternalError, "shm allgather: stale or foreign record");
            }
        }
        for (int r = 0; r < nranks; ++r)
            if (n) std::memcpy(static_cast<uint8_t*>(out) + static_cast<size_t>(r) * n,
                               all.data() + static_cast<size_t>(r) * rec.size() + 8, n);
        b->barrier();  // nobody reads my record any more
    });
}

nimbleResult_t nimbleBootstrapAllgather(const nimbleUniqueId* id, int rank, int nranks, const void* in, size_t n,
                                        void* out) {
    return guarded([&] {
        if (!id || (n && (!in || !out))) throw nb::Error(nimbleInvalidArgument, "bootstrap: null argument");
        auto b = nb::bootstrap_connect(*id, rank, nranks);
        b->allgather(in, n, out);
    });
}

}  // extern "C"
