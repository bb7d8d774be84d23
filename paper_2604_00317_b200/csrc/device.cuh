// Plain-old-data shared by the host runtime and the sm_100a forwarding engine.
//
// Per rank the comm owns two IPC-exported device regions:
//   ctrl    : Ctrl header (posts, done / pulled counters) followed by the ready
//             flags of the staging rings hosted here and the consumed flags of
//             the rings this rank feeds;
//   staging : one ring of `slots` x `pipe_chunk` bytes per ordered pair (s,d)
//             hosted on this rank (used when this rank relays s->d, or, for
//             s->me, when my receive buffer is not registered).
// The flag protocol is the reference's bounded-buffer recurrence
// (proj/src/pipeline.cpp:97-106): chunk k of a
// ring may enter the staging slot k % S only after the forwarder has drained
// chunk k - S (consumed flag), and may leave it only after it has landed
// (ready flag).  Flags carry (epoch << 32 | k + 1) tags, so no reset is needed
// between calls.
#pragma once

#if !defined(__CUDACC__) && !defined(__host__)
#define __host__
#define __device__
#endif

#include <cstdint>

namespace nb {

constexpr int kMaxRanks = 32;
// CommDevice::scratch words: [0] main queue head, [1] CTAs done, then the
// per-peer grant decisions (2 x kMaxRanks), then the push-lane queue head.
constexpr int kScratchPushHead = 2 + 2 * kMaxRanks;
constexpr int kScratchWords = kScratchPushHead + 1;
constexpr int kMaxSlots = 256;
constexpr int kThreads = 512;  // forwarding-engine CTA size

// Low-latency (LL) protocol for small direct pairs: the sender stores 16-byte
// lines {data[0:4], flag, data[4:8], flag} (flag = epoch, low 32 bits) into a
// per-sender slot inside the receiver's ctrl region, which the receiver polls
// and decodes -- no posts, no fences, no completion handshake.  Line 0 carries
// the byte count.  Slots are double-buffered by epoch parity; a sender reuses
// slot e & 1 only after the receiver acknowledged epoch e - 2 (ll_ack).
constexpr uint64_t kLLMaxData = 1ull << 20;                                  // bytes per pair
constexpr uint64_t kLLPiece = 8ull << 10;                                   // bytes per work item (one CTA)
constexpr uint64_t kLLSlotBytes = ((1 + kLLMaxData / 8) * 16 + 255) / 256 * 256;  // header + lines

enum ItemKind : uint8_t {
    kLocal = 0,    // src -> dst, both local absolute addresses
    kPush = 1,     // my send range -> receiver `peer` (zero copy, or its self ring when staged)
    kStage = 2,    // my send range -> ring (me, aux) hosted on relay `peer`
    kForward = 3,  // ring (aux, peer) hosted here -> receiver `peer` (or my own buffer)
    kPull = 4,     // sender `peer`'s registered send range -> my buffer (receiver-driven)
    kLLSend = 5,   // my small segment -> LL slot at receiver `peer` (separate list, see LaunchArgs)
    kLLRecv = 6,   // LL slot of sender `peer` -> my buffer
};

// One unit of the chunk schedule, 32 bytes.
struct Item {
    uint64_t src;    // kLocal/kPush/kStage: absolute local source address; kPull: offset in the segment
    uint64_t dst;    // kLocal/kPull: absolute; kPush/kForward: byte offset inside the pair segment
    uint32_t bytes;  // <= pipe_chunk for ring traffic
    uint8_t kind;
    uint8_t peer;    // kLocal: unused; kPush: receiver; kStage: relay; kForward: final receiver; kPull: sender
    uint16_t aux;    // kStage: final receiver; kForward: original sender
    uint32_t seq;    // chunk index in the ring / flow
    uint32_t pad;
};
static_assert(sizeof(Item) == 32, "Item layout");

// One flow of a rank's chunk schedule (schedule.cpp): item k covers bytes
// [k * chunk, min((k + 1) * chunk, bytes)) of the flow, carries chunk index
// proto.seq + k, and sorts by the key (k + 0.5) / n * scale + phase -- its
// progress fraction (scale 1 except for the parts of a pair built from
// several sends, which share the pair's progress) -- ties going to the larger
// flow, then to the earlier insertion index base + k.  The host merges the
// flows into the item list (schedule.cpp, merge_cuts) or the device does
// (engine.cu, gen_items_kernel) -- identical lists either way.
enum CutFlags : uint32_t { kCutSrc = 1, kCutDst = 2, kCutPull = 4, kCutPushLane = 8 };
struct CutDesc {
    Item proto;             // kind / peer / aux / pad of every item of the flow
    uint64_t src0, dst0;    // item k: src = src0 + k * chunk (kCutSrc), dst = dst0 + k * chunk (kCutDst)
    uint64_t bytes, chunk, n;
    uint64_t src_from_dst;  // kCutPull: src = dst - src_from_dst (offset inside the sender's segment)
    double phase, scale;
    uint32_t base;          // insertion index of item 0
    uint32_t flags;         // CutFlags
};
static_assert(sizeof(CutDesc) == 104, "CutDesc layout");

// Receive posts: where a sender's segment lands (+ a pull request bit).
// Send posts: where my outgoing segment lives, if it is registered.
enum PostMode : uint32_t {
    kPostZeroCopy = 1,
    kPostStaged = 2,
    kPostPullRequest = 0x10,  // receiver asks the sender to let it pull
    kSendRegistered = 1,      // send post: segment readable by the receiver (window win, offset off)
    kSendPlain = 2,           // send post: not registered, the sender pushes
};

// Receiver d publishes, for each sender s, where s's segment lands; sender s
// publishes, for each receiver d, where its outgoing segment lives.
struct Post {
    uint64_t tag;    // epoch of the call this post belongs to
    uint32_t win;    // registered window id (zero copy)
    uint32_t mode;   // PostMode
    uint64_t off;    // byte offset of the pair segment inside the window
    uint64_t bytes;  // expected byte count (checked against the sender's)
};
static_assert(sizeof(Post) == 32, "Post layout");

// A post as published in ctrl: low-latency encoding with the epoch inside
// every 8-byte word, so it is written with plain relaxed stores (no fence) and
// a reader accepts it once all three words carry its epoch:
//   w[0] = epoch32 << 32 | win << 16 | mode,  w[1] = epoch16 << 48 | off,
//   w[2] = epoch16 << 48 | bytes            (off, bytes < 2^48).
// Double-buffered by epoch parity.  A writer that never has to wait for a
// reader can reach epoch e + 2 and overwrite the slot first; the reader then
// sees a newer epoch and infers the outcome (engine.cu, read_post).
struct WirePost {
    uint64_t w[4];
};

// Posts are pushed to their reader, who polls local memory: post_in[e][d] is
// receiver d's post for me (the direct sender), send_post[e][s] is sender s's
// send post for me (the receiver).  post[e][s] is my own copy of my post for
// sender s, read remotely only by relays forwarding s's chunks to me.  Slot
// e & 1 holds epoch e; a slot holding a newer epoch means its writer finished
// epoch e without needing the reader (see read_post in engine.cu).
struct CtrlHeader {
    WirePost post[2][kMaxRanks];       // written by me (the receiver), read by relays
    uint64_t done[kMaxRanks];          // done[w] >= epoch << 32: writer w finished writing into me
    WirePost send_post[2][kMaxRanks];  // send_post[e][s]: pushed by sender s, read by me
    uint64_t pulled[kMaxRanks];        // pulled[d] >= epoch << 32: receiver d finished pulling from me
    WirePost post_in[2][kMaxRanks];    // post_in[e][d]: pushed by receiver d, read by me
    uint64_t ll_ack[kMaxRanks];        // ll_ack[d] = epoch: receiver d finished that launch (its LL slots drained)
};

// Geometry of the flag arrays that follow the header inside ctrl.
struct FlagLayout {
    static constexpr uint64_t header = (sizeof(CtrlHeader) + 255) / 256 * 256;
    // ready flags of ring (s, d) hosted here: [s][d][slot]
    __host__ __device__ static constexpr uint64_t ready_off(int R, int s, int d, int slot) {
        return header + 8ull * ((static_cast<uint64_t>(s) * R + d) * kMaxSlots + slot);
    }
    // consumed flags of ring (me, d) hosted on relay v: [d][v][slot]
    __host__ __device__ static constexpr uint64_t consumed_off(int R, int d, int v, int slot) {
        return header + 8ull * static_cast<uint64_t>(R) * R * kMaxSlots +
               8ull * ((static_cast<uint64_t>(d) * R + v) * kMaxSlots + slot);
    }
    __host__ __device__ static constexpr uint64_t flags_end(int R) { return header + 16ull * R * R * kMaxSlots; }
    // LL slot of sender s hosted here, epoch parity e: [e][s]
    __host__ __device__ static constexpr uint64_t ll_off(int R, int e, int s) {
        return flags_end(R) + (static_cast<uint64_t>(e) * R + s) * kLLSlotBytes;
    }
    // Slot-occupancy counters of ring (s, d) hosted here (NIMBLE_STATS=1): a
    // count of claimed-not-released slots and one word per slot, claimed by
    // the stager after its consumed-flag wait and released by the forwarder
    // before it raises the consumed flag.  The bounded-buffer invariant of
    // the reference (tests/acceptance.cpp:270-288: occupancy <= S) is checked
    // on the device from these.
    __host__ __device__ static constexpr uint64_t occ_count_off(int R, int s, int d) {
        return ll_off(R, 2, 0) + 4ull * ((static_cast<uint64_t>(s) * R + d) * (kMaxSlots + 1));
    }
    __host__ __device__ static constexpr uint64_t bytes(int R) {
        return (occ_count_off(R, R - 1, R) + 255) / 256 * 256;  // one past the last ring
    }
};

// Per-rank device counters (NIMBLE_STATS=1 at comm creation; nimbleCommGetStats).
enum StatKind : int {
    kStatLocal = 0,
    kStatPush = 1,     // by receiver: bytes pushed (zero copy or into its self ring)
    kStatStage = 2,    // by relay: bytes staged into a relay's ring (hop 1)
    kStatForward = 3,  // by final receiver: bytes forwarded out of a ring hosted here (hop 2)
    kStatPull = 4,     // by sender: bytes pulled out of its registered segment
    kStatLLSend = 5,   // by receiver
    kStatLLRecv = 6,   // by sender
    kStatDrain = 7,    // by sender: bytes drained from my self ring (staged receive)
    kStatKinds = 8,
};
struct DeviceStats {
    unsigned long long bytes[kStatKinds][kMaxRanks];
    unsigned long long items[kStatKinds][kMaxRanks];
    unsigned long long occ_max;      // max over my stager claims of the ring's claimed-slot count
    unsigned long long occ_double;   // claims of a slot still held by an undrained chunk (must stay 0)
    unsigned long long occ_claims;   // ring-slot claims made
    unsigned long long pad;
    // host side (filled by nimbleCommGetStats, not by the device): the C ABI's
    // per-call cost -- data-path calls, their total / max wall time, and the
    // plans and schedules built for new matrices (cache misses)
    unsigned long long host_calls, host_ns, host_ns_max;
    unsigned long long plans_built, plan_ns, schedules_built, schedule_ns;
    unsigned long long host_pad;
};

// Comm-lifetime device view (set up once at init / registration).
struct CommDevice {
    int rank, nranks;
    uint8_t* ctrl[kMaxRanks];     // ctrl region of every rank, mapped here
    uint8_t* staging[kMaxRanks];  // staging region of every rank, mapped here
    uint64_t* win_table;          // [win * kMaxRanks + rank] -> mapped window base
    uint32_t nwin;
    uint32_t timeout_ms;
    uint32_t ring_full;           // 1: R x R staging rings (mesh model), 0: R self rings indexed by sender
    uint32_t pad0;
    uint32_t* status;             // host-mapped: [0] error code, [1] detail
    uint64_t* epoch;              // launches completed on this comm (advanced by each launch's last CTA)
    DeviceStats* stats;           // null unless NIMBLE_STATS=1
    uint32_t* scratch;            // [0] queue head, [1] CTAs done, [2, 2+kMaxRanks) grant decisions
                                  // as sender, [2+kMaxRanks, 2+2*kMaxRanks) as receiver (kDecide*)
};

// Device-side schedule generation for a new matrix (engine.cu,
// gen_items_kernel): the flows travel as kernel parameters, so a schedule
// needs no host merge and no upload.  cuts[0, nkeyed) are merged into
// items[0, nitems); cuts[nkeyed, ncuts) are the LL pieces (sends, then
// receives), enumerated in order into ll_items.
constexpr int kMaxGenCuts = 200;
struct GenArgs {
    Item* items;
    Item* ll_items;
    Post* posts;
    Post* send_posts;
    uint32_t ncuts, nkeyed, nitems, nll;
    uint32_t R;
    uint32_t n_push_lane;  // items of the kCutPushLane flows: they come first in `items`
    Post post[kMaxRanks];
    Post send_post[kMaxRanks];
    CutDesc cuts[kMaxGenCuts];
};

constexpr uint64_t kEpochUnknown = ~0ull;

// Per-launch arguments (passed by value as a __grid_constant__ kernel parameter).
struct LaunchArgs {
    const Item* items;
    uint32_t nitems;
    uint32_t slots;        // S
    uint64_t pipe_chunk;   // ring slot bytes
    uint64_t epoch;        // set by the kernel itself from CommDevice::epoch (graph-replay safe)
    const CommDevice* comm;
    const Post* posts;       // [R] my receive posts for this call (device copy)
    const Post* send_posts;  // [R] my send posts for this call (device copy)
    uint64_t recv_direct;             // senders with a direct flow into me
    uint64_t recv_zc;                 // ... whose segment lands in a registered window of mine
    uint64_t pull_req;                // ... from whom I asked to pull
    uint64_t relay_writers;           // relays forwarding into me
    uint64_t push_targets;            // receivers I have kPush items for
    uint64_t write_targets;           // peers whose memory I may write (pushes, relay forwards)
    uint64_t send_bytes[kMaxRanks];   // my outgoing pair sizes (checked against receivers' posts)
    const uint64_t* final_waits;      // pairs (ctrl byte offset of consumed flag, chunk index)
    uint32_t nfinal;
    uint32_t n_ll_send, n_ll_recv;    // LL items: ll_items[0, n_ll_send) sends, then receives
    const Item* ll_items;             // pieces of <= kLLPiece: kLLSend src / kLLRecv dst absolute, peer = the
                                      // other end, seq = piece index, pad = the pair's byte count
    uint64_t ll_senders;              // senders whose LL slot I drain this launch
    uint32_t pull_depth;              // max stages in flight per CTA for a pull (kStages: no cap)
    uint32_t split_signal;            // 1: the last CTA's warp 1 issues the completions owed to peers
                                      // while warp 0 waits and releases the epoch (engine.cu)
    uint32_t tail_items;              // the last tail_items items of the main queue pull one stage at a
                                      // time (a shorter ingress queue at the end: faster acknowledgements)
    uint32_t local_only;              // 1: flagless single-GPU exchange (no ctrl)
    uint64_t* trace;                  // optional globaltimer stamps (NIMBLE_TRACE=1), see kTrace*
    uint32_t n_push_lane;             // items[0, n_push_lane): the push lane (direct pushes of a port that
                                      // declined pulls), taken first by CTAs [0, push_ctas); the rest is
                                      // the main queue, taken by every CTA
    uint32_t push_ctas;
    uint64_t prev_epoch;              // epoch of the previous launch on this comm, when the host knows it
                                      // (kEpochUnknown: after graph captures); the kernel then chains
                                      // on the epoch word instead of griddepcontrol.wait (engine.cu)
};

// Device timeline of one launch (ns, %globaltimer): written when tracing is on.
enum TraceSlot : int {
    kTraceKernelStart = 0,   // min over CTAs: entered the kernel
    kTracePrologueDone = 1,  // CTA 0: posts published
    kTraceFirstItem = 2,     // min over CTAs: first item prepared
    kTraceLastItem = 3,      // max over CTAs: producer out of items
    kTraceCtasDone = 4,      // last CTA arrived at the epilogue
    kTraceSignalled = 5,     // done / pulled published
    kTraceWaited = 6,        // all incoming completions observed
    kTraceFirstCtaDone = 7,  // min over CTAs: first CTA out of work
    kTraceLoopsDoneMax = 8,  // max over CTAs: producer / consumers / signal warp finished
    kTraceFenceDoneMax = 9,  // max over CTAs: completion fence done
    kTraceLoopsDoneMin = 10, // min over CTAs: loops finished
    kTraceEntryMin = 11,     // min over CTAs: entered the kernel, before griddepcontrol.wait (PDL)
    kTracePrevEnd = 12,      // the previous launch's last CTA finished (its last timestamp)
    kTraceSlots = 16,
};
// Per-CTA timeline after the kTraceSlots launch-wide slots (NIMBLE_TRACE=1):
// CTA i owns kTraceSlots + i * kCtaTraceSlots + k.
enum CtaTraceSlot : int {
    kCtaFirstItem = 0,    // producer: first item prepared (ns)
    kCtaQueueEmpty = 1,   // producer: out of items (ns)
    kCtaLoopsDone = 2,    // producer / consumers / signal warp finished (ns)
    kCtaFenceDone = 3,    // completion fence done (ns)
    kCtaRemoteBytes = 4,  // bytes this CTA stored into peer memory (push / stage / forward)
    kCtaOtherBytes = 5,   // bytes it pulled or copied locally
    kCtaTraceSlots = 6,
};
constexpr int kMaxCtaTrace = 160;
constexpr int kTraceWords = kTraceSlots + kMaxCtaTrace * kCtaTraceSlots;
// The trace region holds two such timelines, used by epoch parity (launch e
// writes buffer e & 1 and its last CTA resets buffer (e + 1) & 1 for the
// next launch -- no host operation between launches), then one persistent
// word: the end time of the latest launch.
constexpr int kTraceRegionWords = 2 * kTraceWords + 1;
__host__ __device__ constexpr bool trace_is_min_slot(int k) {
    return k == 0 || k == 2 || k == 7 || k == 10 || k == 11;
}

}  // namespace nb
