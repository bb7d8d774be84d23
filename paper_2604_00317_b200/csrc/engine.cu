// The forwarding engine: one persistent sm_100a kernel per rank per exchange.
//
// Each CTA (512 threads) is warp-specialized:
//   warp 0, lane 0  -- producer: takes 32-byte work items from the rank's chunk
//                      schedule in key order (one atomicAdd per item), resolves
//                      where the bytes go (posts, staging slots), performs the
//                      item's flag waits, and streams the source into a ring of
//                      6 x 32 KB shared-memory stages with TMA bulk copies
//                      (cp.async.bulk global->shared, mbarrier complete_tx);
//                      pulls keep at most 3 stages in flight;
//   warps 1..14     -- consumers: per stage, realign the bytes (source and
//                      destination may be misaligned relative to each other:
//                      two 16-byte shared loads + funnel shifts) and store them
//                      with 16-byte coalesced st.global -- to local HBM, a
//                      peer's registered buffer or a peer's staging slot;
//   warp 15         -- signal warp: raises item-end ready / consumed flags in
//                      item order (system fence + relaxed stores), off the data
//                      path.
// Items are:
//   kLocal   - local copy (self segment, and the 1-GPU emulated exchange);
//   kPush    - direct push into the receiver's registered buffer over NVLink,
//              or into the receiver's self ring when its buffer is unregistered;
//   kStage   - relay hop 1: push into the staging ring hosted on the relay;
//   kForward - relay hop 2 (or the receiver's drain of its self ring):
//              staging slot -> final buffer;
//   kPull    - receiver-driven direct flow: TMA bulk loads straight out of the
//              sender's registered send buffer over NVLink (a receiver asks, a
//              registered sender grants unless its own port is ingress-bound);
//   LL       - small direct pairs (<= ll_max) bypass all of the above: the
//              sender stores data + epoch flags into the receiver's LL slot at
//              kernel start, the receiver polls and decodes at the end.
// Posts (where a segment lands / lives) are pushed by their writer into the
// reader's ctrl region at kernel start; completions are per-pair counters
// (done / pulled) that gain exactly 2^32 per launch: each CTA adds 1 after
// fencing its own writes, the last CTA adds the rest and waits for its peers.
// Ring flags follow the reference's bounded-buffer recurrence
// (proj/src/pipeline.cpp:97-106; device.cuh).  Every wait polls with acquire
// loads and a global-timer timeout that latches an async error instead of
// hanging the GPU.  Kernels are launched with programmatic stream
// serialization: the next exchange's setup overlaps this one's tail, and it
// either chains on this exchange's epoch release (when this exchange is its
// programmatic primary) or waits for its completion (griddepcontrol.wait).
//
// Deadlock freedom: the scheduler sorts every rank's items by a global key
// (chunk progress fraction), every wait targets an item with a strictly
// smaller key, and items are taken in key order -- so the globally smallest
// unfinished item always has its dependencies met.  LL sends wait only for
// the receiver's previous-but-one launch; LL receives only for LL sends.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>

#include "device.cuh"

namespace nb {

namespace {

constexpr int kStageBytes = 32 * 1024;          // bytes of output per stage
constexpr int kStageVecs = kStageBytes / 16;
constexpr int kStages = 6;                      // ring depth
constexpr int kStagePitch = kStageBytes + 128;  // + realignment overhang, 128 B aligned
constexpr int kConsumerWarps = kThreads / 32 - 2;  // warp 0 produces, the last warp signals
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kSignalWarp = kThreads / 32 - 1;
constexpr int kSig = 32;                            // in-flight item-end signals per CTA

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_add_sys(uint64_t* p, uint64_t v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// TMA bulk copy, global -> shared, completion counted on `bar`.
__device__ __forceinline__ void tma_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void st16(void* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__device__ __forceinline__ uint8_t ld_byte(const uint8_t* p, bool coherent) {
    if (!coherent) return __ldg(p);
    unsigned short v;
    asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return static_cast<uint8_t>(v);
}

enum AsyncCode : uint32_t {
    kErrPostTimeout = 1,
    kErrSlotTimeout = 2,
    kErrReadyTimeout = 3,
    kErrDoneTimeout = 4,
    kErrSizeMismatch = 5,
    kErrRelayToStaged = 6,
    kErrFinalTimeout = 7,
    kErrPostLost = 8,  // a post was overwritten in a way the protocol does not allow
    kErrLLTimeout = 9,   // an LL slot never filled (or its receiver never drained the previous one)
    kErrBounds = 10,     // a work item's byte range falls outside its segment or staging slot (scheduler bug)
};

// Latch the first async error of the comm: status[0] = code, status[1] =
// where (peer << 16 | low 16 bits of the epoch), for nimbleCommGetAsyncError.
__device__ __forceinline__ void latch(const CommDevice* c, uint32_t code, uint32_t peer = 0xff, uint64_t epoch = 0) {
    if (atomicCAS(c->status, 0u, code) == 0u) {
        c->status[1] = (peer & 0xffu) << 16 | static_cast<uint32_t>(epoch & 0xffffu);
        __threadfence_system();
    }
}

// Producer-thread wait until *p >= tag; false (and an async error) on timeout
// or when another wait already failed.
__device__ bool wait_ge(const uint64_t* p, uint64_t tag, const CommDevice* c, uint32_t code, uint32_t peer = 0xff) {
    if (ld_acquire(p) >= tag) return true;
    const uint64_t t0 = global_ns();
    const uint64_t limit = static_cast<uint64_t>(c->timeout_ms) * 1000000ull;
    volatile uint32_t* status = c->status;
    for (uint32_t spin = 0;; ++spin) {
        if (ld_acquire(p) >= tag) return true;
        if ((spin & 255) == 255) {
            if (*status != 0) return false;
            if (global_ns() - t0 > limit) {
                latch(c, code, peer, tag >> 32 ? tag >> 32 : tag);
                return false;
            }
        }
        if (spin > 64) __nanosleep(32);
    }
}

__device__ __forceinline__ uint64_t tag_of(uint64_t epoch, uint32_t k) { return (epoch << 32) | (k + 1ull); }

enum StageFlags : uint32_t {
    kTerminate = 1,
    kItemEnd = 2,      // last stage of an item: head/tail bytes + end actions
    kCoherentSrc = 4,  // source written by a peer during this launch (staging)
};

enum EndAction : uint32_t {
    kActRelease1 = 1,  // st.release(flag1, tag1)
    kActRelease2 = 2,  // st.release(flag2, tag2)
};

struct StageDesc {
    uint64_t dst;    // 16-byte aligned destination of the stage's first vector
    uint32_t nvec;   // 16-byte output vectors in the stage
    uint32_t shift;  // source misalignment (0..15) of the body
    uint32_t flags;
    uint32_t action;
    uint64_t head_src, head_dst, tail_src, tail_dst;
    uint32_t head_n, tail_n;
    uint32_t sig;  // signal-ring entry of the item's end actions
    // filled by prepare() for the producer's use only (copied into the SigDesc)
    uint64_t* flag1;
    uint64_t tag1;
    uint64_t* flag2;
    uint64_t tag2;
    uint32_t* occ;  // NIMBLE_STATS: the drained ring's claimed-slot count (slot word at occ + 1 + occ_slot)
    uint32_t occ_slot;
};

// Item-end actions handed from the consumers to the signal warp, which does
// the system fence and the flag releases off the data path.
struct SigDesc {
    uint32_t action, terminate;
    uint64_t* flag1;
    uint64_t tag1;
    uint64_t* flag2;
    uint64_t tag2;
    uint32_t* occ;
    uint32_t occ_slot;
};

struct SharedState {
    uint64_t full[kStages];
    uint64_t empty[kStages];
    StageDesc desc[kStages];
    uint64_t sig_full[kSig];   // consumers (one arrive per warp) -> signal warp
    uint64_t sig_empty[kSig];  // signal warp -> producer
    SigDesc sig[kSig];
    uint64_t seg_base[kMaxRanks * kMaxRanks];  // (receiver, sender) -> resolved segment base
    uint64_t seg_bytes[kMaxRanks * kMaxRanks]; // (receiver, sender) -> the segment's byte count (bounds checks)
    uint32_t seg_mode[kMaxRanks * kMaxRanks];  // 0 = unresolved
    uint64_t send_base[kMaxRanks];             // sender -> its registered send segment (pull)
    uint32_t send_mode[kMaxRanks];             // 0 = unresolved
    uint32_t remote_writes;                    // this CTA stored into peer memory
};

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

struct PostView {
    uint32_t mode, win;
    uint64_t off, bytes;
};

enum PostRead { kPostFailed, kPostOk, kPostAdvanced };

// Wait for this epoch's post at p and decode it.  kPostFailed (async error)
// on timeout.  With `may_advance`, a slot already holding a NEWER epoch
// returns kPostAdvanced: the writer finished this epoch and the next one
// without waiting for me, which the protocol allows in exactly one way per
// post kind (resolve / resolve_send say which) -- so the overwritten post's
// content is implied and the reader does not wait for a post that will never
// come back.
__device__ PostRead read_post(const WirePost* p, uint64_t epoch, const CommDevice* c, PostView& out,
                              bool may_advance) {
    const uint64_t e32 = epoch & 0xffffffffull, e16 = epoch & 0xffffull;
    const uint64_t t0 = global_ns();
    const uint64_t limit = static_cast<uint64_t>(c->timeout_ms) * 1000000ull;
    for (uint32_t spin = 0;; ++spin) {
        const uint64_t w0 = ld_acquire(&p->w[0]);
        if ((w0 >> 32) == e32) {
            const uint64_t w1 = ld_relaxed(&p->w[1]), w2 = ld_relaxed(&p->w[2]);
            if ((w1 >> 48) == e16 && (w2 >> 48) == e16) {
                out.mode = static_cast<uint32_t>(w0 & 0xffff);
                out.win = static_cast<uint32_t>((w0 >> 16) & 0xffff);
                out.off = w1 & 0xffffffffffffull;
                out.bytes = w2 & 0xffffffffffffull;
                return kPostOk;
            }
        } else if (may_advance && static_cast<int32_t>(static_cast<uint32_t>(w0 >> 32) - static_cast<uint32_t>(e32)) > 0) {
            return kPostAdvanced;
        }
        if ((spin & 255) == 255) {
            if (*reinterpret_cast<volatile uint32_t*>(c->status) != 0) return kPostFailed;
            if (global_ns() - t0 > limit) {
                latch(c, kErrPostTimeout, 0xff, epoch);
                return kPostFailed;
            }
        }
        if (spin > 64) __nanosleep(32);
    }
}

__device__ __forceinline__ void write_post(WirePost* p, uint64_t epoch, const Post& v) {
    const uint64_t e16 = (epoch & 0xffffull) << 48;
    st_relaxed(&p->w[1], e16 | (v.off & 0xffffffffffffull));
    st_relaxed(&p->w[2], e16 | (v.bytes & 0xffffffffffffull));
    st_relaxed(&p->w[0], (epoch & 0xffffffffull) << 32 | (static_cast<uint64_t>(v.win & 0xffff) << 16) |
                             (v.mode & 0xffff));
}

enum Decide : uint32_t { kDecidePull = 1, kDecidePush = 2 };  // per-launch grant records (scratch)

// Resolve receiver d's post for sender s (producer thread): the direct
// sender reads the copy d pushed into its own ctrl, a relay reads d's.
__device__ bool resolve(SharedState& sh, const LaunchArgs& a, int d, int s) {
    const int key = d * kMaxRanks + s;
    if (sh.seg_mode[key]) return true;
    const CommDevice* c = a.comm;
    const bool direct = s == c->rank;
    PostView v;
    const PostRead r = direct
        ? read_post(&reinterpret_cast<const CtrlHeader*>(c->ctrl[s])->post_in[a.epoch & 1][d], a.epoch, c, v, true)
        : read_post(&reinterpret_cast<const CtrlHeader*>(c->ctrl[d])->post[a.epoch & 1][s], a.epoch, c, v, false);
    if (r == kPostFailed) return false;
    if (r == kPostAdvanced) {
        // d got past this epoch without waiting for me, so it did not take my
        // push: it pulled my segment, which needs my send window registered.
        if (a.send_posts[d].mode != kSendRegistered) {
            atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrPostLost));
            return false;
        }
        sh.seg_base[key] = 0;
        sh.seg_bytes[key] = a.send_bytes[d];
        sh.seg_mode[key] = kPostZeroCopy | kPostPullRequest;
        c->scratch[2 + d] = kDecidePull;
        return true;
    }
    const uint32_t mode = v.mode, win = v.win;
    const uint64_t off = v.off;
    if (direct) {  // my own outgoing segment: sizes must agree end to end
        const uint64_t expect = v.bytes;
        if (expect != a.send_bytes[d]) {
            atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrSizeMismatch));
            return false;
        }
    }
    sh.seg_base[key] = (mode & 0xf) == kPostZeroCopy ? c->win_table[win * kMaxRanks + d] + off : 0;
    sh.seg_bytes[key] = v.bytes;
    sh.seg_mode[key] = mode;
    if (direct)  // record, for the epilogue, whether d pulls my segment or takes pushes
        c->scratch[2 + d] = ((mode & kPostPullRequest) && a.send_posts[d].mode == kSendRegistered) ? kDecidePull
                                                                                                    : kDecidePush;
    return true;
}

// Sender s's send post for me (the receiver), cached per CTA.  False on timeout.
__device__ bool resolve_send(SharedState& sh, const LaunchArgs& a, int s) {
    if (sh.send_mode[s]) return true;
    const CommDevice* c = a.comm;
    PostView v;
    const PostRead r =
        read_post(&reinterpret_cast<const CtrlHeader*>(c->ctrl[c->rank])->send_post[a.epoch & 1][s], a.epoch, c, v, true);
    if (r == kPostFailed) return false;
    if (r == kPostAdvanced) {
        // s got past this epoch without waiting for my pull: it pushed (declined).
        v.mode = kSendPlain;
        v.win = 0;
        v.off = 0;
    }
    const uint32_t mode = v.mode, win = v.win;
    const uint64_t off = v.off;
    c->scratch[2 + kMaxRanks + s] = mode == kSendRegistered ? kDecidePull : kDecidePush;
    sh.send_base[s] = mode == kSendRegistered ? c->win_table[win * kMaxRanks + s] + off : 0;
    sh.send_mode[s] = mode;
    asm volatile("fence.proxy.async.global;" ::: "memory");  // generic -> async proxy (TMA reads)
    return true;
}

// Does receiver d pull my segment instead of me pushing it?  (d asked, and
// my send segment for d is registered.)  Needs d's receive post resolved.
__device__ __forceinline__ bool pull_granted_to(const SharedState& sh, const LaunchArgs& a, int d) {
    const int me = a.comm->rank;
    return (sh.seg_mode[d * kMaxRanks + me] & kPostPullRequest) && a.send_posts[d].mode == kSendRegistered;
}

__device__ __forceinline__ uint8_t* ring_slot(const LaunchArgs& a, int host, int s, int d, uint32_t seq) {
    const int R = a.comm->nranks;
    // ring (s, d) hosted on `host`: R x R rings under the mesh model, else only
    // self rings (host == d), indexed by sender
    const uint64_t ring = a.comm->ring_full ? static_cast<uint64_t>(s) * R + d : static_cast<uint64_t>(s);
    return a.comm->staging[host] + (ring * a.slots + seq % a.slots) * a.pipe_chunk;
}

__device__ __forceinline__ uint64_t* ctrl_flag(const LaunchArgs& a, int rank, uint64_t off) {
    return reinterpret_cast<uint64_t*>(a.comm->ctrl[rank] + off);
}

// NIMBLE_STATS: stager side of the slot-occupancy check (FlagLayout).  Runs
// after the consumed-flag acquire, so the forwarder's release of chunk
// seq - S (done before it raised that flag) is visible here.
__device__ void claim_slot(const CommDevice* c, int host, int s, int d, uint32_t slot, uint32_t seq) {
    auto* cnt = reinterpret_cast<unsigned int*>(c->ctrl[host] + FlagLayout::occ_count_off(c->nranks, s, d));
    const unsigned int prev = atomicExch_system(cnt + 1 + slot, seq + 1);
    const unsigned int occ = atomicAdd_system(cnt, 1u) + 1;
    if (prev) atomicAdd(&c->stats->occ_double, 1ull);
    atomicAdd(&c->stats->occ_claims, 1ull);
    atomicMax(&c->stats->occ_max, static_cast<unsigned long long>(occ));
}

__device__ __forceinline__ void count_item(const CommDevice* c, int kind, int peer, uint64_t bytes) {
    atomicAdd(&c->stats->bytes[kind][peer], static_cast<unsigned long long>(bytes));
    atomicAdd(&c->stats->items[kind][peer], 1ull);
}

enum Prep { kGo, kSkip };

// Every item's byte range must lie inside the segment (or staging slot) it
// addresses -- true by construction of the schedule; checked anyway, on
// every item, because a violation would write another rank's memory.  A few
// integer compares per item (items are 8-64 KiB).
__device__ __forceinline__ bool in_bounds(const CommDevice* c, uint64_t off, uint32_t bytes, uint64_t limit) {
    if (off + bytes <= limit) return true;
    atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrBounds));
    return false;
}

// Producer: the item's source, destination and end-of-item actions.  kSkip
// when the item has nothing to do (pull granted / declined) or a wait failed
// (the error is latched in the status word).
__device__ Prep prepare(SharedState& sh, const LaunchArgs& a, const Item& it, uint64_t& src, uint64_t& dst,
                        StageDesc& end, bool& coherent) {
    const CommDevice* c = a.comm;
    const int me = c->rank, R = c->nranks;
    src = it.src;
    dst = it.dst;
    coherent = false;
    end.action = 0;
    if (it.kind == kLocal) return kGo;
    if (it.kind == kPull) {  // my direct flow from sender s, if s granted the pull
        const int s = it.peer;
        if (!resolve_send(sh, a, s)) return kSkip;
        if (sh.send_mode[s] != kSendRegistered) return kSkip;  // declined: s pushes instead
        if (!in_bounds(c, it.src, it.bytes, a.posts[s].bytes)) return kSkip;  // inside s's segment for me
        src = sh.send_base[s] + it.src;  // pulled[] is counted once per CTA (epilogue)
        return kGo;
    }
    if (it.kind == kPush || it.kind == kStage) {
        const int host = it.peer;  // receiver (push) or relay (stage)
        const int d = it.kind == kPush ? it.peer : it.aux;
        if (it.kind == kPush) {
            if (!resolve(sh, a, d, me)) return kSkip;
            if (pull_granted_to(sh, a, d)) return kSkip;  // d pulls this range itself
            if (!in_bounds(c, it.dst, it.bytes, a.send_bytes[d])) return kSkip;  // inside my segment for d
            if ((sh.seg_mode[d * kMaxRanks + me] & 0xf) == kPostZeroCopy) {
                dst = sh.seg_base[d * kMaxRanks + me] + it.dst;  // done[] is counted once per CTA (epilogue)
                return kGo;
            }
        }
        if (!in_bounds(c, 0, it.bytes, a.pipe_chunk)) return kSkip;  // one staging slot
        const uint32_t slot = it.seq % a.slots;
        if (it.seq >= a.slots &&
            !wait_ge(ctrl_flag(a, me, FlagLayout::consumed_off(R, d, host, slot)), tag_of(a.epoch, it.seq - a.slots), c,
                     kErrSlotTimeout))
            return kSkip;
        if (c->stats) claim_slot(c, host, me, d, slot, it.seq);
        dst = reinterpret_cast<uint64_t>(ring_slot(a, host, me, d, it.seq));
        end.action = kActRelease1;  // chunk landed in the slot: raise its ready flag
        end.flag1 = ctrl_flag(a, host, FlagLayout::ready_off(R, me, d, slot));
        end.tag1 = tag_of(a.epoch, it.seq);
        return kGo;
    }
    // kForward: ring (s, d) hosted here -> receiver d
    const int s = it.aux, d = it.peer;
    if (d == me && ((a.pull_req >> s) & 1)) {  // my self ring is idle if s granted my pull
        if (!resolve_send(sh, a, s)) return kSkip;
        if (sh.send_mode[s] == kSendRegistered) return kSkip;
    }
    const uint32_t slot = it.seq % a.slots;
    if (!wait_ge(ctrl_flag(a, me, FlagLayout::ready_off(R, s, d, slot)), tag_of(a.epoch, it.seq), c, kErrReadyTimeout))
        return kSkip;
    asm volatile("fence.proxy.async.global;" ::: "memory");  // peer-written slot, read by TMA
    coherent = true;
    src = reinterpret_cast<uint64_t>(ring_slot(a, me, s, d, it.seq));
    end.action = kActRelease2;  // the slot is drained: hand it back to the stager
    end.flag2 = ctrl_flag(a, s, FlagLayout::consumed_off(R, d, me, slot));
    end.tag2 = tag_of(a.epoch, it.seq);
    end.occ = c->stats ? reinterpret_cast<uint32_t*>(c->ctrl[me] + FlagLayout::occ_count_off(R, s, d)) : nullptr;
    end.occ_slot = slot;
    if (d == me) {
        dst = a.posts[s].off + it.dst;  // staged self receive: absolute local address
        return kGo;
    }
    if (!resolve(sh, a, d, s)) return kSkip;
    if ((sh.seg_mode[d * kMaxRanks + s] & 0xf) != kPostZeroCopy) {
        atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrRelayToStaged));
        return kSkip;
    }
    if (!in_bounds(c, it.dst, it.bytes, sh.seg_bytes[d * kMaxRanks + s])) return kSkip;  // inside d's segment for s
    dst = sh.seg_base[d * kMaxRanks + s] + it.dst;
    return kGo;
}

__device__ __forceinline__ void trace_min(const LaunchArgs& a, int slot) {
    if (a.trace) atomicMin(reinterpret_cast<unsigned long long*>(a.trace + slot), global_ns());
}
__device__ __forceinline__ void trace_max(const LaunchArgs& a, int slot) {
    if (a.trace) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + slot), global_ns());
}

// ---- low-latency (LL) protocol for small direct pairs (device.cuh, kLLMaxData) ----

__device__ __forceinline__ void st_ll(uint4* p, uint32_t lo, uint32_t hi, uint32_t flag) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(lo), "r"(flag), "r"(hi),
                 "r"(flag)
                 : "memory");
}

__device__ __forceinline__ uint4 ld_ll(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

// Bytes [off, off + n) of p (n <= 8) as a little-endian word; any alignment.
__device__ __forceinline__ uint64_t load_upto8(const uint8_t* p, uint32_t n) {
    if (n == 8 && (reinterpret_cast<uintptr_t>(p) & 7) == 0) return *reinterpret_cast<const uint64_t*>(p);
    uint64_t v = 0;
    for (uint32_t i = 0; i < n; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
    return v;
}

__device__ __forceinline__ void store_upto8(uint8_t* p, uint64_t v, uint32_t n) {
    if (n == 8 && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
        *reinterpret_cast<uint64_t*>(p) = v;
        return;
    }
    for (uint32_t i = 0; i < n; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}

// Every CTA, all threads, at kernel start: my small segments straight into
// the receivers' LL slots.  The only wait is for the slot's previous use
// (epoch - 2) to have been drained, which is almost always long done.
__device__ void ll_send_all(const LaunchArgs& a) {
    const CommDevice* c = a.comm;
    const int me = c->rank, R = c->nranks;
    const uint32_t flag = static_cast<uint32_t>(a.epoch);
    __shared__ uint32_t ok;
    for (uint32_t j = blockIdx.x; j < a.n_ll_send; j += gridDim.x) {
        const Item it = a.ll_items[j];
        const int d = it.peer;
        if (threadIdx.x == 0) {
            const CtrlHeader* h = reinterpret_cast<const CtrlHeader*>(c->ctrl[me]);
            ok = a.epoch <= 2 || wait_ge(&h->ll_ack[d], a.epoch - 2, c, kErrLLTimeout, static_cast<uint32_t>(d));
        }
        __syncthreads();
        if (ok) {
            // line 0: the pair's byte count (written by piece 0); piece p's data
            // byte b sits in line 1 + (p * kLLPiece + b) / 8
            uint4* slot = reinterpret_cast<uint4*>(c->ctrl[d] + FlagLayout::ll_off(R, static_cast<int>(a.epoch & 1), me));
            uint4* lines0 = slot + 1 + it.seq * (kLLPiece / 8);
            const uint8_t* src = reinterpret_cast<const uint8_t*>(it.src);
            const uint32_t n = it.bytes, lines = (n + 7) / 8;
            if (it.seq == 0 && threadIdx.x == 0) st_ll(slot, it.pad, ~it.pad, flag);
            if (threadIdx.x == 0 && c->stats) count_item(c, kStatLLSend, d, it.bytes);
            for (uint32_t k = threadIdx.x; k < lines; k += blockDim.x) {
                const uint32_t off = 8 * k, m = n - off < 8 ? n - off : 8;
                const uint64_t v = load_upto8(src + off, m);
                st_ll(lines0 + k, static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32), flag);
            }
        }
        __syncthreads();
    }
}

// Every CTA, all threads, after its forwarding work: poll my LL slots and
// decode them into the receive buffer.  A line is valid once both of its
// 8-byte halves carry this epoch's flag.
__device__ void ll_recv_all(const LaunchArgs& a) {
    const CommDevice* c = a.comm;
    const int me = c->rank, R = c->nranks;
    const uint32_t flag = static_cast<uint32_t>(a.epoch);
    const uint64_t limit = static_cast<uint64_t>(c->timeout_ms) * 1000000ull;
    volatile uint32_t* status = c->status;
    for (uint32_t j = blockIdx.x; j < a.n_ll_recv; j += gridDim.x) {
        const Item it = a.ll_items[a.n_ll_send + j];
        const int s = it.peer;
        const uint4* slot =
            reinterpret_cast<const uint4*>(c->ctrl[me] + FlagLayout::ll_off(R, static_cast<int>(a.epoch & 1), s));
        const uint4* lines0 = slot + 1 + it.seq * (kLLPiece / 8);
        uint8_t* dst = reinterpret_cast<uint8_t*>(it.dst);
        const uint32_t n = it.bytes, lines = (n + 7) / 8;
        if (threadIdx.x == 0 && c->stats) count_item(c, kStatLLRecv, s, n);
        // thread slot k = lines is piece 0's header check (line 0)
        const uint32_t last = it.seq == 0 ? lines : lines - 1;
        for (uint32_t k = threadIdx.x; k <= last; k += blockDim.x) {
            const uint4* line = k == lines ? slot : lines0 + k;
            uint4 v = ld_ll(line);
            if (v.y != flag || v.w != flag) {
                const uint64_t t0 = global_ns();
                for (uint32_t spin = 0;; ++spin) {
                    v = ld_ll(line);
                    if (v.y == flag && v.w == flag) break;
                    if ((spin & 255) == 255) {
                        if (*status != 0) break;
                        if (global_ns() - t0 > limit) {
                            if (atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrLLTimeout)) == 0u) {
                                // what the line held: its two flag words, and which line / piece
                                c->status[1] = (0x80u | static_cast<uint32_t>(s)) << 16 |
                                               static_cast<uint32_t>(a.epoch & 0xffffu);
                                c->status[2] = v.y;
                                c->status[3] = v.w;
                                c->status[4] = k;
                                c->status[5] = it.seq;
                                __threadfence_system();
                            }
                            break;
                        }
                    }
                    if (spin > 16) __nanosleep(64);  // thousands of pollers: keep L2 free for the incoming lines
                }
                if (v.y != flag || v.w != flag) break;  // error latched
            }
            if (k == lines) {
                if (v.x != it.pad || v.z != ~it.pad) atomicCAS(c->status, 0u, static_cast<uint32_t>(kErrSizeMismatch));
            } else {
                const uint32_t off = 8 * k, m = n - off < 8 ? n - off : 8;
                store_upto8(dst + off, static_cast<uint64_t>(v.x) | static_cast<uint64_t>(v.z) << 32, m);
            }
        }
    }
}

__device__ void produce(SharedState& sh, uint8_t* stages, const LaunchArgs& a) {
    uint32_t* scratch = a.comm->scratch;
    uint32_t cnt = 0, nsig = 0;
    auto next_sig = [&]() {
        const uint32_t j = nsig % kSig;
        if (nsig >= kSig) mbar_wait(&sh.sig_empty[j], ((nsig / kSig) - 1) & 1);
        ++nsig;
        return j;
    };
    bool first = true;
    uint64_t remote_bytes = 0, other_bytes = 0;
    uint64_t* ctr = a.trace && blockIdx.x < kMaxCtaTrace ? a.trace + kTraceSlots + blockIdx.x * kCtaTraceSlots : nullptr;
    auto next_slot = [&](uint32_t& slot) {
        slot = cnt % kStages;
        if (cnt >= kStages) mbar_wait(&sh.empty[slot], ((cnt / kStages) - 1) & 1);
    };
    // The push lane first (CTAs [0, push_ctas)), then the main queue.  Each
    // queue is in key order, so the deadlock-freedom argument holds per queue:
    // a lane push waits only for posts and for its receiver's drain of slot
    // k - S (the receiver's main queue), never for this rank's main queue.
    const bool lane = blockIdx.x < a.push_ctas;
    for (uint32_t* qhead = lane ? &scratch[kScratchPushHead] : &scratch[0];;) {
        const bool main_q = qhead == &scratch[0];
        const uint32_t qbase = main_q ? a.n_push_lane : 0;
        const uint32_t qn = main_q ? a.nitems - a.n_push_lane : a.n_push_lane;
        const uint32_t index = atomicAdd(qhead, 1u);
        if (index >= qn) {
            if (main_q) break;
            qhead = &scratch[0];
            continue;
        }
        const Item it = a.items[qbase + index];
        uint64_t src, dst;
        StageDesc end{};
        bool coherent = false;
        if (prepare(sh, a, it, src, dst, end, coherent) != kGo) continue;
        const bool remote = it.kind == kPush || it.kind == kStage || (it.kind == kForward && it.peer != a.comm->rank);
        if (remote) sh.remote_writes = 1;
        if (ctr) (remote ? remote_bytes : other_bytes) += it.bytes;
        if (first) {
            trace_min(a, kTraceFirstItem);
            if (ctr) ctr[kCtaFirstItem] = global_ns();
            first = false;
        }
        uint32_t sig = 0;
        if (end.action) {
            sig = next_sig();
            SigDesc& sd = sh.sig[sig];
            sd.action = end.action;
            sd.terminate = 0;
            sd.flag1 = end.flag1;
            sd.tag1 = end.tag1;
            sd.flag2 = end.flag2;
            sd.tag2 = end.tag2;
            sd.occ = end.occ;
            sd.occ_slot = end.occ_slot;
        }
        if (a.comm->stats) {
            const int me = a.comm->rank;
            const int kind = it.kind == kForward ? (it.peer == me ? kStatDrain : kStatForward) : it.kind;
            count_item(a.comm, kind, kind == kStatDrain ? it.aux : it.peer, it.bytes);
        }
        // head: bytes until the destination is 16-byte aligned
        uint64_t n = it.bytes;
        uint32_t head = static_cast<uint32_t>((16 - (dst & 15)) & 15);
        if (head > n) head = static_cast<uint32_t>(n);
        const uint64_t bsrc = src + head, bdst = dst + head;
        n -= head;
        const uint64_t n16 = n >> 4;
        const uint32_t tail = static_cast<uint32_t>(n & 15);
        const uint32_t shift = static_cast<uint32_t>(bsrc & 15);
        const uint64_t src_al = bsrc - shift;
        const uint64_t src_al_end = (bsrc + (n16 << 4) + 15) & ~15ull;
        const uint64_t nstages = n16 ? (n16 + kStageVecs - 1) / kStageVecs : 1;
        for (uint64_t k = 0; k < nstages; ++k) {
            uint32_t slot;
            next_slot(slot);
            // Remote (NVLink) sources need far less in flight than HBM copies
            // (~16 KB per CTA covers the link's latency-bandwidth product): cap
            // a pull at pull_depth outstanding stages so the drain at the end
            // of the exchange stays short.
            const uint32_t depth = main_q && index + a.tail_items >= qn ? 1u : a.pull_depth;
            if (it.kind == kPull && depth < kStages && cnt >= depth) {
                const uint32_t j = cnt - depth;
                mbar_wait(&sh.empty[j % kStages], (j / kStages) & 1);
            }
            StageDesc& ds = sh.desc[slot];
            const uint64_t v0 = k * kStageVecs;
            const uint32_t nvec = static_cast<uint32_t>(n16 > v0 ? (n16 - v0 < kStageVecs ? n16 - v0 : kStageVecs) : 0);
            ds.dst = bdst + (v0 << 4);
            ds.nvec = nvec;
            ds.shift = shift;
            ds.flags = coherent ? kCoherentSrc : 0;
            if (k + 1 == nstages) {
                ds.flags |= kItemEnd;
                ds.action = end.action;
                ds.head_src = src;
                ds.head_dst = dst;
                ds.head_n = head;
                ds.tail_src = bsrc + (n16 << 4);
                ds.tail_dst = bdst + (n16 << 4);
                ds.tail_n = tail;
                ds.sig = sig;
            }
            uint32_t bytes = 0;
            if (nvec) {
                const uint64_t from = src_al + (v0 << 4);
                const uint64_t want = (static_cast<uint64_t>(nvec) << 4) + (shift ? 16 : 0);
                bytes = static_cast<uint32_t>(src_al_end - from < want ? src_al_end - from : want);
            }
            if (bytes) {
                mbar_arrive_tx(&sh.full[slot], bytes);
                tma_load(stages + slot * kStagePitch, reinterpret_cast<const void*>(src_al + (v0 << 4)), bytes,
                         &sh.full[slot]);
            } else {
                mbar_arrive(&sh.full[slot]);
            }
            ++cnt;
        }
    }
    trace_max(a, kTraceLastItem);
    if (ctr) {
        ctr[kCtaQueueEmpty] = global_ns();
        ctr[kCtaRemoteBytes] = remote_bytes;
        ctr[kCtaOtherBytes] = other_bytes;
    }
    uint32_t slot;
    next_slot(slot);
    sh.desc[slot].flags = kTerminate;
    mbar_arrive(&sh.full[slot]);
    const uint32_t j = next_sig();  // and stop the signal warp
    sh.sig[j].terminate = 1;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&sh.sig_full[j])),
                 "r"(kConsumerWarps)
                 : "memory");
}

// Signal warp (lane 0): item-end flag releases, in item order, one fence per
// batch of completed items.
__device__ void signal_loop(SharedState& sh) {
    for (uint32_t n = 0;; ++n) {
        const uint32_t j = n % kSig;
        mbar_wait(&sh.sig_full[j], (n / kSig) & 1);
        const SigDesc sd = sh.sig[j];
        if (sd.terminate) break;
        if (sd.occ) {  // NIMBLE_STATS: release the drained slot before handing it back
            atomicExch_system(sd.occ + 1 + sd.occ_slot, 0u);
            atomicSub_system(sd.occ, 1u);
        }
        asm volatile("fence.acq_rel.sys;" ::: "memory");  // the item's bytes before its flag
        if (sd.action & kActRelease1) st_relaxed(sd.flag1, sd.tag1);
        if (sd.action & kActRelease2) st_relaxed(sd.flag2, sd.tag2);
        mbar_arrive(&sh.sig_empty[j]);
    }
}

template <int q>
__device__ __forceinline__ void realign_store(const uint4* buf, uint8_t* out, uint32_t nvec, uint32_t bits, int ct) {
    for (uint32_t j = ct; j < nvec; j += kConsumers) {
        const uint4 x = buf[j], y = buf[j + 1];
        const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
        uint4 o;
        o.x = __funnelshift_r(w[q + 0], w[q + 1], bits);
        o.y = __funnelshift_r(w[q + 1], w[q + 2], bits);
        o.z = __funnelshift_r(w[q + 2], w[q + 3], bits);
        o.w = __funnelshift_r(w[q + 3], w[q + 4], bits);
        st16(out + 16ull * j, o);
    }
}

__device__ void consume(SharedState& sh, const uint8_t* stages, const LaunchArgs& a) {
    const int ct = threadIdx.x - 32;  // consumer thread index
    const int lane = threadIdx.x & 31;
    (void)a;
    for (uint32_t cnt = 0;; ++cnt) {
        const uint32_t slot = cnt % kStages;
        mbar_wait(&sh.full[slot], (cnt / kStages) & 1);
        const StageDesc ds = sh.desc[slot];
        if (ds.flags & kTerminate) break;
        const uint4* buf = reinterpret_cast<const uint4*>(stages + slot * kStagePitch);
        uint8_t* out = reinterpret_cast<uint8_t*>(ds.dst);
        const uint32_t bits = (ds.shift & 3) * 8;
        switch (ds.shift ? 1 + (ds.shift >> 2) : 0) {  // uniform across the CTA
        case 0:
            for (uint32_t j = ct; j < ds.nvec; j += kConsumers) st16(out + 16ull * j, buf[j]);
            break;
        case 1: realign_store<0>(buf, out, ds.nvec, bits, ct); break;
        case 2: realign_store<1>(buf, out, ds.nvec, bits, ct); break;
        case 3: realign_store<2>(buf, out, ds.nvec, bits, ct); break;
        default: realign_store<3>(buf, out, ds.nvec, bits, ct); break;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[slot]);
        if (ds.flags & kItemEnd) {
            const bool coh = ds.flags & kCoherentSrc;
            if (ct < static_cast<int>(ds.head_n))
                reinterpret_cast<uint8_t*>(ds.head_dst)[ct] = ld_byte(reinterpret_cast<const uint8_t*>(ds.head_src) + ct, coh);
            if (ct >= 32 && ct < 32 + static_cast<int>(ds.tail_n))
                reinterpret_cast<uint8_t*>(ds.tail_dst)[ct - 32] =
                    ld_byte(reinterpret_cast<const uint8_t*>(ds.tail_src) + (ct - 32), coh);
            if (ds.action) {  // hand the item to the signal warp (no fence on the data path)
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.sig_full[ds.sig]);
            }
        }
    }
}

constexpr size_t kEngineSmem = sizeof(SharedState) + 128 + static_cast<size_t>(kStages) * kStagePitch;

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) exchange_kernel(const __grid_constant__ LaunchArgs args) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    SharedState& sh = *reinterpret_cast<SharedState*>(smem_raw);
    // The launch's epoch comes from device memory, not the host: a launch
    // captured in a CUDA graph and replayed gets a fresh epoch every time.
    // Launched with programmatic stream serialization: this grid may start
    // while the previous exchange on the stream is still finishing.  Until
    // the chaining decision below, only this CTA's shared memory and the
    // comm's immutable view are touched.
    __shared__ LaunchArgs a;
    if (threadIdx.x == 0) a = args;
    uint8_t* stages = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw + sizeof(SharedState)) + 127) & ~static_cast<uintptr_t>(127));
    const CommDevice* c = args.comm;  // the parameter, not the shared copy (not yet synced)
    const int tid = threadIdx.x;

    for (int i = tid; i < kMaxRanks * kMaxRanks; i += kThreads) sh.seg_mode[i] = 0;
    for (int i = tid; i < kMaxRanks; i += kThreads) sh.send_mode[i] = 0;
    if (tid == 0) sh.remote_writes = 0;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sh.full[s], 1);
            mbar_init(&sh.empty[s], kConsumerWarps);
        }
        for (int j = 0; j < kSig; ++j) {
            mbar_init(&sh.sig_full[j], kConsumerWarps);
            mbar_init(&sh.sig_empty[j], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint64_t entry_ns = args.trace && tid == 0 ? global_ns() : 0;
    // Chaining to the previous exchange of this comm.  When the host knows
    // that launch's epoch, wait for its last CTA's release of the epoch word
    // (written after it reset the shared scratch and trace state): this grid
    // (a programmatic dependent) then starts ~5 us before the previous grid's
    // completion would release griddepcontrol.wait.  Otherwise (launches
    // replayed from CUDA graphs), wait for the previous grid's completion.
    // The host allows this only when the previous launch of the library on
    // this stream was this comm's previous exchange.  A CTA that finds that
    // exchange still running (epoch word behind) knows it is the primary of
    // this launch -- any other work on the stream would have had to wait for
    // its completion -- and chains on the epoch word; one that finds it done
    // does the ordinary griddepcontrol.wait (cheap then), so work a user
    // enqueued in between is always waited for.
    __shared__ uint32_t need_wait, early;
    if (tid == 0) {
        need_wait = 1;
        early = 0;
        if (!args.local_only && args.prev_epoch != kEpochUnknown &&
            ld_acquire(c->epoch) < args.prev_epoch) {
            need_wait = 0;
            early = 1;
            a.epoch = args.prev_epoch + 1;
        }
    }
    __syncthreads();
    const int me = c->rank, R = c->nranks;
    // Prologue: publish where each sender's segment lands in my buffer, and
    // where my outgoing segments live.  A chained launch does it before the
    // previous exchange has released the epoch: that exchange is this
    // launch's primary (so no other work touched the buffers in between) and
    // all its CTAs are past their data movement (they triggered this
    // launch), so the posts for the next epoch can go out now -- peers start
    // moving data into / out of my buffers ~a completion latency earlier.
    auto publish_posts = [&]() {
        if (a.local_only || blockIdx.x != 0 || tid >= 2 * R) return;
        const bool send_side = tid >= R;
        const int peer = send_side ? tid - R : tid;
        const Post p = send_side ? a.send_posts[peer] : a.posts[peer];
        if (!p.tag) return;
        // pushed to the reader (it polls local memory); my own copy of a
        // receive post serves relays
        CtrlHeader* ph = reinterpret_cast<CtrlHeader*>(c->ctrl[peer]);
        const int e = static_cast<int>(a.epoch & 1);
        if (send_side) {
            write_post(&ph->send_post[e][me], a.epoch, p);
        } else {
            write_post(&ph->post_in[e][me], a.epoch, p);
            write_post(&reinterpret_cast<CtrlHeader*>(c->ctrl[me])->post[e][peer], a.epoch, p);
        }
    };
    if (early) publish_posts();
    if (tid == 0 && early)
        for (uint32_t spin = 0; ld_acquire(c->epoch) < args.prev_epoch; ++spin)
            if (spin > 64) __nanosleep(64);
    if (need_wait) asm volatile("griddepcontrol.wait;" ::: "memory");  // prior grids complete, their writes visible
    if (tid == 0) {
        if (!early) a.epoch = a.local_only ? 0 : *reinterpret_cast<volatile uint64_t*>(c->epoch) + 1;
        if (a.trace) {  // this launch's timeline: buffer epoch & 1 (see kTraceRegionWords)
            a.trace = args.trace + (a.epoch & 1) * kTraceWords;
            atomicMin(reinterpret_cast<unsigned long long*>(a.trace + kTraceEntryMin), entry_ns);
            if (blockIdx.x == 0) a.trace[kTracePrevEnd] = args.trace[2 * kTraceWords];
        }
        trace_min(a, kTraceKernelStart);
    }
    __syncthreads();
    uint32_t* scratch = c->scratch;
    if (!early) publish_posts();
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) trace_max(a, kTracePrologueDone);
    if (a.n_ll_send) ll_send_all(a);

    const int warp = tid / 32;
    if (warp == 0) {
        if (tid == 0) produce(sh, stages, a);
    } else if (warp == kSignalWarp) {
        if ((tid & 31) == 0) signal_loop(sh);
    } else {
        consume(sh, stages, a);
    }
    __syncthreads();
    if (tid == 0) {
        trace_max(a, kTraceLoopsDoneMax);
        trace_min(a, kTraceLoopsDoneMin);
        if (a.trace && blockIdx.x < kMaxCtaTrace) a.trace[kTraceSlots + blockIdx.x * kCtaTraceSlots + kCtaLoopsDone] = global_ns();
    }
    if (a.n_ll_recv) ll_recv_all(a);
    if (tid == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // next exchange may start launching

    // Epilogue.  done[me] / pulled[me] at every peer are per-pair counters that
    // gain exactly 2^32 per launch, so "epoch e complete" is counter >= e << 32:
    // each CTA, once its own writes are fenced, adds 1 for every peer it may
    // have written into (done) or pulled from (pulled); the last CTA adds the
    // rest (2^32 - grid, or 2^32 for a peer this launch does not touch).  The
    // sum can only reach the threshold after every CTA's add has landed, and
    // every add is issued after that CTA's fence -- so the last CTA needs no
    // second system fence.  It then waits for everyone else's completions --
    // one warp, lane p handling peer p -- and resets the per-launch scratch for
    // the next stream-ordered launch.
    __shared__ uint32_t last_cta;
    if (tid < 32) {
        if (tid == 0) {
            // this CTA's peer writes before its completion adds (pulls and local
            // copies only read remote memory: a GPU-scope fence will do)
            // release (not sequentially consistent) fences: all the adds below need
            if (sh.remote_writes) asm volatile("fence.acq_rel.sys;" ::: "memory");
            else asm volatile("fence.acq_rel.gpu;" ::: "memory");
            trace_min(a, kTraceFirstCtaDone);
            trace_max(a, kTraceFenceDoneMax);
            if (a.trace && blockIdx.x < kMaxCtaTrace) a.trace[kTraceSlots + blockIdx.x * kCtaTraceSlots + kCtaFenceDone] = global_ns();
        }
        __syncwarp();
        if (!a.local_only && tid < R) {
            CtrlHeader* ph = reinterpret_cast<CtrlHeader*>(c->ctrl[tid]);
            if ((a.write_targets >> tid) & 1) red_add_sys(&ph->done[me], 1);
            if ((a.pull_req >> tid) & 1) red_add_sys(&ph->pulled[me], 1);
        }
        __syncwarp();
        if (tid == 0) last_cta = atomicAdd(&scratch[1], 1u) + 1 == gridDim.x;
    }
    __syncthreads();
    // The completions this launch owes its peers: done / pulled counters
    // topped up to exactly 2^32 per peer, and the LL acknowledgement (this
    // launch's LL slots are drained: acknowledged to every peer, LL sender now
    // or not, so a sender's wait for epoch - 2 never depends on which pairs
    // were small back then).  Issued by warp 1 while warp 0 waits for the
    // peers' completions and releases the epoch: warp 0's release fence then
    // does not wait for these remote writes' acknowledgements (which queue
    // behind a saturated ingress), and nothing warp 0 waits for depends on
    // them being issued first by warp 0 (NIMBLE_SPLIT_SIGNAL=0: warp 0 issues
    // them itself, before its waits).
    auto signal_peers = [&](int lane) {
        const uint64_t full = 1ull << 32;
        if (lane < R) {
            CtrlHeader* ph = reinterpret_cast<CtrlHeader*>(c->ctrl[lane]);
            red_add_sys(&ph->done[me], ((a.write_targets >> lane) & 1) ? full - gridDim.x : full);
            red_add_sys(&ph->pulled[me], ((a.pull_req >> lane) & 1) ? full - gridDim.x : full);
            st_relaxed(&ph->ll_ack[me], a.epoch);
        }
        __syncwarp();
        if (lane == 0) trace_max(a, kTraceSignalled);
    };
    if (last_cta && a.split_signal && !a.local_only && tid >= 32 && tid < 64) signal_peers(tid - 32);
    if (last_cta && tid < 32) {
        const int lane = tid;
        if (lane == 0) trace_max(a, kTraceCtasDone);
        if (!a.local_only) {
            const uint64_t done_tag = a.epoch << 32;
            if (!a.split_signal) signal_peers(lane);
            for (uint32_t i = lane; i < a.nfinal; i += 32)  // relayed chunks drained from their rings
                wait_ge(reinterpret_cast<const uint64_t*>(c->ctrl[me] + a.final_waits[2 * i]),
                        tag_of(a.epoch, static_cast<uint32_t>(a.final_waits[2 * i + 1])), c, kErrFinalTimeout);
            if (lane < R) {
                const int w = lane;
                const CtrlHeader* h = reinterpret_cast<const CtrlHeader*>(c->ctrl[me]);
                const uint32_t* decide = scratch + 2;
                bool need_done = (a.relay_writers >> w) & 1;
                if (((a.recv_direct >> w) & 1) && ((a.recv_zc >> w) & 1))  // w pushed in place unless I pulled
                    need_done |= !(((a.pull_req >> w) & 1) && decide[kMaxRanks + w] == kDecidePull);
                if (need_done) wait_ge(&h->done[w], done_tag, c, kErrDoneTimeout, static_cast<uint32_t>(w));
                if (((a.push_targets >> w) & 1) && decide[w] == kDecidePull)  // w pulled my segment
                    wait_ge(&h->pulled[w], done_tag, c, kErrDoneTimeout, 0x80u | static_cast<uint32_t>(w));
            }
            __syncwarp();
        }
        if (lane < R) scratch[2 + lane] = scratch[2 + kMaxRanks + lane] = 0;
        __syncwarp();
        if (lane == 0) {
            trace_max(a, kTraceWaited);
            scratch[0] = 0;
            scratch[1] = 0;
            scratch[kScratchPushHead] = 0;
        }
    }
    if (last_cta) {
        if (a.trace) {  // reset the other timeline for the next launch, stamp this one's end
            __syncthreads();
            uint64_t* next = args.trace + ((a.epoch + 1) & 1) * kTraceWords;
            for (int k = tid; k < kTraceWords; k += kThreads)
                next[k] = k < kTraceSlots && trace_is_min_slot(k) ? ~0ull : 0;
            __syncthreads();
            if (tid == 0) args.trace[2 * kTraceWords] = global_ns();
        }
        // Last: publish the epoch.  The next exchange of this comm (possibly
        // already resident, see the chaining above) starts when it sees it,
        // so everything this launch shares with it -- scratch, trace -- is
        // reset before this release.
        if (tid == 0 && !a.local_only) {
            __threadfence();
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(c->epoch), "l"(a.epoch) : "memory");
        }
    }
}

// ---- device-side schedule generation (new matrices: no host merge, no upload) ----
//
// Item (f, k) of the keyed flows lands at position
//     sum over flows g of #{k' : (g, k') before (f, k)}
// in the merged list, with `before` the host merge's order (schedule.cpp):
// key (k + 0.5) / n + phase, then the larger flow, then insertion index.  A
// flow's keys increase with k, so each count is a prefix length, found from
// a closed-form guess and a few exact comparisons.  Keys are computed with
// the same IEEE operations as the host (correctly rounded divide and add,
// no contraction), so the list is the host's, item for item.

__device__ __forceinline__ double gen_key(const CutDesc& f, uint64_t k) {
    return __dadd_rn(__dmul_rn(__ddiv_rn(static_cast<double>(k) + 0.5, static_cast<double>(f.n)), f.scale), f.phase);
}

__device__ __forceinline__ bool gen_before(const CutDesc& a, uint64_t ka, double keya, const CutDesc& b, uint64_t kb,
                                           double keyb) {
    if (keya != keyb) return keya < keyb;
    if (a.bytes != b.bytes) return a.bytes > b.bytes;
    return a.base + ka < b.base + kb;
}

__device__ __forceinline__ Item gen_item(const CutDesc& f, uint64_t k) {
    Item it = f.proto;
    const uint64_t off = k * f.chunk;
    it.src = (f.flags & kCutSrc) ? f.src0 + off : 0;
    it.dst = (f.flags & kCutDst) ? f.dst0 + off : 0;
    it.bytes = static_cast<uint32_t>(f.chunk < f.bytes - off ? f.chunk : f.bytes - off);
    it.seq = f.proto.seq + static_cast<uint32_t>(k);
    if (f.flags & kCutPull) it.src = it.dst - f.src_from_dst;
    return it;
}

__global__ void __launch_bounds__(256) gen_items_kernel(const __grid_constant__ GenArgs g) {
    __shared__ CutDesc cuts[kMaxGenCuts];
    for (uint32_t i = threadIdx.x; i < g.ncuts; i += blockDim.x) cuts[i] = g.cuts[i];
    if (blockIdx.x == 0)
        for (uint32_t r = threadIdx.x; r < g.R; r += blockDim.x) {
            g.posts[r] = g.post[r];
            g.send_posts[r] = g.send_post[r];
        }
    __syncthreads();
    const uint32_t total = g.nitems + g.nll;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < total; j += gridDim.x * blockDim.x) {
        // the flow holding insertion index j (bases ascend within each group)
        const bool ll = j >= g.nitems;
        const uint32_t idx = ll ? j - g.nitems : j;
        uint32_t lo = ll ? g.nkeyed : 0, hi = ll ? g.ncuts : g.nkeyed;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (cuts[mid].base <= idx) lo = mid;
            else hi = mid;
        }
        const CutDesc& f = cuts[lo];
        const uint64_t k = idx - f.base;
        if (ll) {  // LL pieces keep their order: base is the slot in ll_items
            g.ll_items[idx] = gen_item(f, k);
            continue;
        }
        const double key = gen_key(f, k);
        // position within the item's queue: the push lane first, then the rest
        const uint32_t lane = f.flags & kCutPushLane;
        uint64_t pos = lane ? 0 : g.n_push_lane;
        for (uint32_t h = 0; h < g.nkeyed; ++h) {
            const CutDesc& c = cuts[h];
            if ((c.flags & kCutPushLane) != lane) continue;
            if (h == lo) {
                pos += k;
                continue;
            }
            // guess: k' with (k' + 0.5) / n * scale + phase < key, then settle exactly
            const double x = (key - c.phase) / c.scale * static_cast<double>(c.n) - 0.5;
            int64_t q = x <= 0.0 ? 0 : (x >= static_cast<double>(c.n) ? static_cast<int64_t>(c.n) : static_cast<int64_t>(ceil(x)));
            while (q < static_cast<int64_t>(c.n) && gen_before(c, q, gen_key(c, q), f, k, key)) ++q;
            while (q > 0 && !gen_before(c, q - 1, gen_key(c, q - 1), f, k, key)) --q;
            pos += static_cast<uint64_t>(q);
        }
        g.items[pos] = gen_item(f, k);
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

// Library kernel launches in this process, any stream (comm.cpp: an
// exchange chains on its predecessor's epoch only when nothing else of the
// library was launched since, see LaunchArgs::prev_epoch).
std::atomic<uint64_t> g_launch_seq{0};

cudaError_t prepare_engine(int dev) {
    static std::mutex mu;
    static bool done[64] = {};
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(mu);
    if (done[dev]) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(exchange_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kEngineSmem));
    // Load every kernel of the library now (CUDA loads modules lazily, on a
    // function's first launch, and a module load waits for the device's
    // running kernels -- on a device hosting several ranks, peer engines that
    // may be spinning on this rank's next launch).
    cudaFuncAttributes fa;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, gen_items_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fill_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, check_kernel);
    if (e == cudaSuccess) done[dev] = true;
    return e;
}

cudaError_t launch_exchange(const LaunchArgs& args, int ctas, cudaStream_t stream, bool pdl) {
    g_launch_seq.fetch_add(1, std::memory_order_relaxed);
    // Opt in to > 48 KB of dynamic shared memory, once per device for the
    // process (prepare_engine, called at comm creation): changing a kernel's
    // shared-memory configuration can serialize kernels of other streams, and
    // a rank sharing the device may be spinning on a peer's flags right now.
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaError_t e = prepare_engine(dev); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(ctas));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kEngineSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap with the previous exchange's tail
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, exchange_kernel, args);
}

cudaError_t launch_gen(const GenArgs& g, cudaStream_t st) {
    g_launch_seq.fetch_add(1, std::memory_order_relaxed);
    const uint32_t total = g.nitems + g.nll;
    if (!total && !g.R) return cudaSuccess;
    uint32_t blocks = (total + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 1184) blocks = 1184;  // 8 x 148 SMs, grid-stride beyond
    gen_items_kernel<<<blocks, 256, 0, st>>>(g);
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
    g_launch_seq.fetch_add(1, std::memory_order_relaxed);
    if (!n) return cudaSuccess;
    fill_kernel<<<grid_for((n >> 3) + 2), 256, 0, st>>>(static_cast<uint8_t*>(buf), first, n, payload_key(seed, s, d));
    return cudaGetLastError();
}

cudaError_t launch_check(const void* buf, uint64_t first, uint64_t n, uint64_t seed, int s, int d, uint64_t* bad,
                         cudaStream_t st) {
    g_launch_seq.fetch_add(1, std::memory_order_relaxed);
    if (!n) return cudaSuccess;
    check_kernel<<<grid_for((n >> 3) + 2), 256, 0, st>>>(static_cast<const uint8_t*>(buf), first, n,
                                                         payload_key(seed, s, d),
                                                         reinterpret_cast<unsigned long long*>(bad));
    return cudaGetLastError();
}

}  // namespace nb
