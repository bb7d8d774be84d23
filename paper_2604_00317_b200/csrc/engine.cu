// The forwarding engine: one persistent sm_100a kernel per rank per exchange.
//
// Every CTA (512 threads) pulls 32-byte work items from the rank's chunk
// schedule in order (one atomicAdd per item) and moves the item's bytes with
// 16-byte vector loads/stores, 8 in flight per thread (64 KiB per CTA
// iteration).  Items are:
//   kLocal   - local copy (self segment, and the 1-GPU emulated exchange);
//   kPush    - direct push into the receiver's registered buffer over NVLink
//              (peer stores into IPC-mapped memory), or into the receiver's
//              self ring when its buffer is not registered;
//   kStage   - relay hop 1: push into the staging ring hosted on the relay;
//   kForward - relay hop 2 (or the receiver's own drain of its self ring):
//              staging slot -> final buffer.
// Flags follow proj/src/pipeline.cpp:97-106 (see device.cuh).  Waits are
// polled by one thread per CTA with acquire loads and a global-timer timeout
// that raises an async error instead of hanging the GPU.
//
// Deadlock freedom: the scheduler sorts every rank's items by a global key
// (chunk progress fraction), every wait targets an item with a strictly
// smaller key, and CTAs take items in key order -- so the globally smallest
// unfinished item always has its dependencies met.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"

namespace nb {

namespace {

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <bool kStreaming>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
    uint4 v;
    if (kStreaming)  // read-only user buffer: no L1 allocation
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p));
    else  // staging written by a peer during this kernel: L2 only
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p));
    return v;
}

__device__ __forceinline__ void st16(uint4* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

template <bool kStreaming>
__device__ __forceinline__ uint8_t ld1(const uint8_t* p) {
    if (kStreaming) return __ldg(p);
    unsigned short v;
    asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return static_cast<uint8_t>(v);
}

constexpr int kUnroll = 8;

// Co-aligned body: src and dst both 16-byte aligned.
template <bool kStreaming>
__device__ __forceinline__ void copy_aligned(const uint4* __restrict__ s, uint4* __restrict__ d, uint64_t n16) {
    uint64_t i = threadIdx.x;
    for (; i + (kUnroll - 1) * kThreads < n16; i += kUnroll * kThreads) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ld16<kStreaming>(s + i + u * kThreads);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) st16(d + i + u * kThreads, v[u]);
    }
    for (; i < n16; i += kThreads) st16(d + i, ld16<kStreaming>(s + i));
}

// dst 16-byte aligned, src off by `sh` (1..15) bytes: two aligned source
// vectors per output vector, realigned with funnel shifts (q = word shift).
template <bool kStreaming, int q>
__device__ __forceinline__ void copy_shifted_q(const uint4* __restrict__ s_al, uint4* __restrict__ d,
                                               uint64_t n16, uint32_t bits) {
    for (uint64_t i = threadIdx.x; i < n16; i += kThreads) {
        const uint4 a = ld16<kStreaming>(s_al + i);
        const uint4 b = ld16<kStreaming>(s_al + i + 1);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint4 o;
        o.x = __funnelshift_r(w[q + 0], w[q + 1], bits);
        o.y = __funnelshift_r(w[q + 1], w[q + 2], bits);
        o.z = __funnelshift_r(w[q + 2], w[q + 3], bits);
        o.w = __funnelshift_r(w[q + 3], w[q + 4], bits);
        st16(d + i, o);
    }
}

// CTA-wide copy of n bytes with arbitrary alignment.
template <bool kStreaming>
__device__ void cta_copy(const uint8_t* __restrict__ s, uint8_t* __restrict__ d, uint64_t n) {
    uint64_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
    if (head > n) head = n;
    if (threadIdx.x < head) d[threadIdx.x] = ld1<kStreaming>(s + threadIdx.x);
    s += head;
    d += head;
    n -= head;
    const uint64_t n16 = n >> 4;
    const uint32_t sh = reinterpret_cast<uintptr_t>(s) & 15;
    if (sh == 0) {
        copy_aligned<kStreaming>(reinterpret_cast<const uint4*>(s), reinterpret_cast<uint4*>(d), n16);
    } else if (n16) {
        const uint4* s_al = reinterpret_cast<const uint4*>(s - sh);
        uint4* dv = reinterpret_cast<uint4*>(d);
        const uint32_t bits = (sh & 3) * 8;
        switch (sh >> 2) {
        case 0: copy_shifted_q<kStreaming, 0>(s_al, dv, n16, bits); break;
        case 1: copy_shifted_q<kStreaming, 1>(s_al, dv, n16, bits); break;
        case 2: copy_shifted_q<kStreaming, 2>(s_al, dv, n16, bits); break;
        default: copy_shifted_q<kStreaming, 3>(s_al, dv, n16, bits); break;
        }
    }
    const uint64_t done = n16 << 4;
    if (threadIdx.x < n - done) d[done + threadIdx.x] = ld1<kStreaming>(s + done + threadIdx.x);
}

// Single-thread wait until *p >= tag; false (and an async error) on timeout
// or when another wait already failed.
__device__ bool wait_ge(const uint64_t* p, uint64_t tag, const CommDevice* c, uint32_t code) {
    if (ld_acquire(p) >= tag) return true;
    const uint64_t t0 = global_ns();
    const uint64_t limit = static_cast<uint64_t>(c->timeout_ms) * 1000000ull;
    volatile uint32_t* status = c->status;
    for (uint32_t spin = 0;; ++spin) {
        if (ld_acquire(p) >= tag) return true;
        if ((spin & 255) == 255) {
            if (*status != 0) return false;
            if (global_ns() - t0 > limit) {
                atomicCAS(c->status, 0u, code);
                return false;
            }
        }
        if (spin > 64) __nanosleep(32);
    }
}

__device__ __forceinline__ uint64_t tag_of(uint64_t epoch, uint32_t k) { return (epoch << 32) | (k + 1ull); }

enum AsyncCode : uint32_t {
    kErrPostTimeout = 1,
    kErrSlotTimeout = 2,
    kErrReadyTimeout = 3,
    kErrDoneTimeout = 4,
    kErrSizeMismatch = 5,
    kErrRelayToStaged = 6,
    kErrFinalTimeout = 7,
};

struct SharedState {
    uint64_t seg_base[kMaxRanks * kMaxRanks];  // (receiver, sender) -> resolved segment base, 0 = unresolved
    uint32_t seg_mode[kMaxRanks * kMaxRanks];
    Item item;
    uint64_t src, dst;
    uint32_t index;
    uint32_t ok;
};

// Resolve receiver d's post for sender s (thread 0 only).
__device__ bool resolve(SharedState& sh, const LaunchArgs& a, int d, int s) {
    const int key = d * kMaxRanks + s;
    if (sh.seg_mode[key]) return true;
    const CommDevice* c = a.comm;
    const Post* p = reinterpret_cast<const Post*>(c->ctrl[d]) + s;
    if (!wait_ge(&p->tag, a.epoch, c, kErrPostTimeout)) return false;
    const uint32_t mode = *reinterpret_cast<const volatile uint32_t*>(&p->mode);
    const uint32_t win = *reinterpret_cast<const volatile uint32_t*>(&p->win);
    const uint64_t off = *reinterpret_cast<const volatile uint64_t*>(&p->off);
    if (s == c->rank) {  // my own outgoing segment: sizes must agree end to end
        const uint64_t expect = *reinterpret_cast<const volatile uint64_t*>(&p->bytes);
        if (expect != a.send_bytes[d]) {
            atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrSizeMismatch));
            return false;
        }
    }
    sh.seg_base[key] = mode == kPostZeroCopy ? c->win_table[win * kMaxRanks + d] + off : 0;
    sh.seg_mode[key] = mode;
    return true;
}

__device__ __forceinline__ uint8_t* ring_slot(const LaunchArgs& a, int host, int s, int d, uint32_t seq) {
    const int R = a.comm->nranks;
    const uint64_t ring = static_cast<uint64_t>(s) * R + d;
    return a.comm->staging[host] + (ring * a.slots + seq % a.slots) * a.pipe_chunk;
}

// After a CTA finished an item that wrote into receiver d's memory: count it
// and, on the receiver's last item from this rank, publish done[me] = epoch.
__device__ void count_write(SharedState& sh, const LaunchArgs& a, int d, uint32_t* counters) {
    const int me = a.comm->rank;
    uint32_t target = a.fwd_items[d];
    if (a.push_items[d]) {  // my pushes count only if d takes them in place
        if (!resolve(sh, a, d, me)) return;
        if (sh.seg_mode[d * kMaxRanks + me] == kPostZeroCopy) target += a.push_items[d];
    }
    __threadfence_system();
    const uint32_t prev = atomicAdd(&counters[d], 1u);
    if (prev + 1 == target) {
        CtrlHeader* h = reinterpret_cast<CtrlHeader*>(a.comm->ctrl[d]);
        st_release(&h->done[me], a.epoch);
    }
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) exchange_kernel(const __grid_constant__ LaunchArgs a) {
    __shared__ SharedState sh;
    const CommDevice* c = a.comm;
    const int tid = threadIdx.x;
    uint32_t* scratch = c->scratch;
    uint32_t* counters = scratch + 2;
    const int me = c->rank, R = c->nranks;

    for (int i = tid; i < kMaxRanks * kMaxRanks; i += kThreads) sh.seg_mode[i] = 0;
    // Prologue: publish where each sender's segment lands in my buffer.
    if (!a.local_only && blockIdx.x == 0 && tid < R) {
        const Post p = a.posts[tid];
        if (p.tag) {
            Post* mine = reinterpret_cast<CtrlHeader*>(c->ctrl[me])->post + tid;
            mine->win = p.win;
            mine->mode = p.mode;
            mine->off = p.off;
            mine->bytes = p.bytes;
            st_release(&mine->tag, p.tag);
        }
    }
    __syncthreads();

    for (;;) {
        if (tid == 0) {
            sh.index = atomicAdd(&scratch[0], 1u);
            sh.ok = 1;
            if (sh.index < a.nitems) {
                const Item it = a.items[sh.index];
                sh.item = it;
                uint64_t src = it.src, dst = it.dst;
                if (it.kind == kPush || it.kind == kStage) {
                    const int host = it.peer;  // receiver (push) or relay (stage)
                    const int d = it.kind == kPush ? it.peer : it.aux;
                    bool staged = it.kind == kStage;
                    if (it.kind == kPush) {
                        sh.ok = resolve(sh, a, d, me);
                        staged = sh.ok && sh.seg_mode[d * kMaxRanks + me] == kPostStaged;
                        if (sh.ok && !staged) dst = sh.seg_base[d * kMaxRanks + me] + it.dst;
                    }
                    if (sh.ok && staged) {
                        if (it.seq >= a.slots) {
                            const uint64_t* f = reinterpret_cast<const uint64_t*>(
                                c->ctrl[me] + FlagLayout::consumed_off(R, d, host, it.seq % a.slots));
                            sh.ok = wait_ge(f, tag_of(a.epoch, it.seq - a.slots), c, kErrSlotTimeout);
                        }
                        dst = reinterpret_cast<uint64_t>(ring_slot(a, host, me, d, it.seq));
                    }
                } else if (it.kind == kForward) {
                    const int s = it.aux, d = it.peer;
                    const uint64_t* f =
                        reinterpret_cast<const uint64_t*>(c->ctrl[me] + FlagLayout::ready_off(R, s, d, it.seq % a.slots));
                    sh.ok = wait_ge(f, tag_of(a.epoch, it.seq), c, kErrReadyTimeout);
                    src = reinterpret_cast<uint64_t>(ring_slot(a, me, s, d, it.seq));
                    if (d == me) {
                        dst = a.posts[s].off + it.dst;  // staged self receive: absolute local address
                    } else if (sh.ok) {
                        sh.ok = resolve(sh, a, d, s);
                        if (sh.ok && sh.seg_mode[d * kMaxRanks + s] != kPostZeroCopy) {
                            atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrRelayToStaged));
                            sh.ok = 0;
                        }
                        if (sh.ok) dst = sh.seg_base[d * kMaxRanks + s] + it.dst;
                    }
                }
                sh.src = src;
                sh.dst = dst;
            }
        }
        __syncthreads();
        if (sh.index >= a.nitems) break;
        const Item it = sh.item;
        if (sh.ok) {
            if (it.kind == kForward)
                cta_copy<false>(reinterpret_cast<const uint8_t*>(sh.src), reinterpret_cast<uint8_t*>(sh.dst), it.bytes);
            else
                cta_copy<true>(reinterpret_cast<const uint8_t*>(sh.src), reinterpret_cast<uint8_t*>(sh.dst), it.bytes);
        }
        __syncthreads();
        if (tid == 0 && sh.ok) {
            if (it.kind == kPush || it.kind == kStage) {
                const int d = it.kind == kPush ? it.peer : it.aux;
                const bool staged = it.kind == kStage || sh.seg_mode[d * kMaxRanks + me] == kPostStaged;
                if (staged) {  // chunk landed in the ring slot: raise its ready flag
                    __threadfence_system();
                    uint64_t* f = reinterpret_cast<uint64_t*>(c->ctrl[it.peer] +
                                                              FlagLayout::ready_off(R, me, d, it.seq % a.slots));
                    st_release(f, tag_of(a.epoch, it.seq));
                } else {
                    count_write(sh, a, d, counters);
                }
            } else if (it.kind == kForward) {
                const int s = it.aux, d = it.peer;
                // the slot's bytes are all read (stores issued): hand it back to the stager
                uint64_t* f = reinterpret_cast<uint64_t*>(c->ctrl[s] + FlagLayout::consumed_off(R, d, me, it.seq % a.slots));
                if (d != me) count_write(sh, a, d, counters);
                st_release(f, tag_of(a.epoch, it.seq));
            }
        }
    }

    // Epilogue: the last CTA out waits for (a) my staged chunks to be drained
    // from their rings, (b) every writer into my buffer to report done; then
    // resets the per-launch scratch for the next stream-ordered launch.
    if (tid == 0) {
        __threadfence();
        const uint32_t arrived = atomicAdd(&scratch[1], 1u);
        if (arrived + 1 == gridDim.x) {
            if (!a.local_only) {
                for (uint32_t i = 0; i < a.nfinal; ++i)
                    wait_ge(reinterpret_cast<const uint64_t*>(c->ctrl[me] + a.final_waits[2 * i]), tag_of(a.epoch, static_cast<uint32_t>(a.final_waits[2 * i + 1])), c, kErrFinalTimeout);
                const CtrlHeader* h = reinterpret_cast<const CtrlHeader*>(c->ctrl[me]);
                for (int w = 0; w < R; ++w)
                    if ((a.expect_done >> w) & 1) wait_ge(&h->done[w], a.epoch, c, kErrDoneTimeout);
            }
            for (int d = 0; d < R; ++d) counters[d] = 0;
            scratch[0] = 0;
            __threadfence();
            scratch[1] = 0;
        }
    }
}

// ---- payload fill / check (test and bench helpers) ----

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fill_kernel(uint8_t* buf, uint64_t first, uint64_t n, uint64_t key) {
    const uint64_t w0 = first >> 3, w1 = (first + n + 7) >> 3;
    for (uint64_t w = w0 + blockIdx.x * blockDim.x + threadIdx.x; w < w1; w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t v = splitmix64(key ^ w);
        const uint64_t lo = w << 3;
        uint8_t* p = buf + (lo - first);  // may point before buf for the first word
        if (lo >= first && lo + 8 <= first + n && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
            *reinterpret_cast<uint64_t*>(p) = v;
        } else {
            for (int b = 0; b < 8; ++b) {
                const uint64_t at = lo + b;
                if (at >= first && at < first + n) buf[at - first] = static_cast<uint8_t>(v >> (8 * b));
            }
        }
    }
}

__global__ void check_kernel(const uint8_t* buf, uint64_t first, uint64_t n, uint64_t key, unsigned long long* bad) {
    const uint64_t w0 = first >> 3, w1 = (first + n + 7) >> 3;
    unsigned long long mine = 0;
    for (uint64_t w = w0 + blockIdx.x * blockDim.x + threadIdx.x; w < w1; w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t v = splitmix64(key ^ w);
        const uint64_t lo = w << 3;
        const uint8_t* p = buf + (lo - first);
        if (lo >= first && lo + 8 <= first + n && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
            const uint64_t got = *reinterpret_cast<const uint64_t*>(p);
            if (got != v)
                for (int b = 0; b < 8; ++b) mine += ((got ^ v) >> (8 * b) & 0xff) != 0;
        } else {
            for (int b = 0; b < 8; ++b) {
                const uint64_t at = lo + b;
                if (at >= first && at < first + n) mine += buf[at - first] != static_cast<uint8_t>(v >> (8 * b));
            }
        }
    }
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(bad, mine);
}

// ---- host-side launchers (called from the comm runtime) ----

cudaError_t launch_exchange(const LaunchArgs& args, int ctas, cudaStream_t stream) {
    exchange_kernel<<<ctas, kThreads, 0, stream>>>(args);
    return cudaGetLastError();
}

static int grid_for(uint64_t words) {
    uint64_t g = (words + 255) / 256;
    return static_cast<int>(g < 4096 ? (g ? g : 1) : 4096);
}

uint64_t payload_key(uint64_t seed, int s, int d) {
    return seed ^ (static_cast<uint64_t>(s) << 48) ^ (static_cast<uint64_t>(d) << 40);
}

cudaError_t launch_fill(void* buf, uint64_t first, uint64_t n, uint64_t seed, int s, int d, cudaStream_t st) {
    if (!n) return cudaSuccess;
    fill_kernel<<<grid_for((n >> 3) + 2), 256, 0, st>>>(static_cast<uint8_t*>(buf), first, n, payload_key(seed, s, d));
    return cudaGetLastError();
}

cudaError_t launch_check(const void* buf, uint64_t first, uint64_t n, uint64_t seed, int s, int d, uint64_t* bad,
                         cudaStream_t st) {
    if (!n) return cudaSuccess;
    check_kernel<<<grid_for((n >> 3) + 2), 256, 0, st>>>(static_cast<const uint8_t*>(buf), first, n,
                                                         payload_key(seed, s, d),
                                                         reinterpret_cast<unsigned long long*>(bad));
    return cudaGetLastError();
}

}  // namespace nb
