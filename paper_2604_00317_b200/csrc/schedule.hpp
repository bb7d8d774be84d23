// The chunk scheduler: turns the replicated plan plus this rank's buffers into
// the rank's ordered work-item list for the forwarding engine.
//
// Byte-range convention (the reference defines
// none): a pair's flows, in candidate order (direct first, then relays in
// ascending GPU order), take consecutive ranges of the pair segment; every
// ring-borne flow is cut into pipe_chunk units with a short tail
// (proj/src/pipeline.cpp:85-91), chunk k riding staging slot k % S.
//
// Order: each item gets the key (k + 0.5) / n of its flow (progress fraction)
// plus a tiny phase offset for hop 2, so all flows advance in proportion and
// finish together (the hot destination's port is fed from t = 0 to the end),
// and every cross-rank wait points at a strictly smaller key -- the engine's
// deadlock-freedom argument (engine.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "device.cuh"
#include "planner.hpp"

namespace nb {

struct RankBuffers {
    int R = 0, me = 0;
    std::vector<uint64_t> send_ptr, send_bytes;  // [R] my outgoing segments
    std::vector<uint64_t> recv_ptr, recv_bytes;  // [R] my incoming segments
    std::vector<Post> recv_post;                 // [R] mode/win/off per sender (tag != 0: present)
    std::vector<Post> send_post;                 // [R] registered window of each outgoing segment
    bool pull = false;                           // ask senders to let me pull my direct flows
    // [R] pairs built from several group operations: (ptr, bytes) per
    // operation, in issue order (empty or one entry: a plain segment)
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> send_parts, recv_parts;
};

struct Schedule {
    std::vector<CutDesc> cuts;     // the keyed flows (merged into the item list)
    std::vector<CutDesc> ll_cuts;  // LL sends, then LL receives (pieces enumerated in order)
    uint32_t nitems = 0;           // items of the keyed flows
    uint32_t n_push_lane = 0;      // of which in the push lane (kCutPushLane flows; first in `items`)
    uint64_t push_lane_bytes = 0, main_bytes = 0;
    std::vector<Item> items;       // materialize(): the merged list (host)
    std::vector<Item> ll_items;    // materialize(): LL sends, then LL receives (engine: LaunchArgs::ll_items)
    uint32_t n_ll_send = 0, n_ll_recv = 0;
    uint64_t ll_senders = 0;
    std::vector<Post> posts;
    std::vector<uint64_t> final_waits;  // (ctrl byte offset, chunk index) pairs
    std::vector<Post> send_posts;
    uint32_t push_items[kMaxRanks] = {};
    uint32_t fwd_items[kMaxRanks] = {};
    uint32_t pull_items[kMaxRanks] = {};
    uint64_t recv_direct = 0, recv_zc = 0, pull_req = 0, relay_writers = 0, push_targets = 0, write_targets = 0;
    int relay_flows = 0;
    uint64_t moved_bytes = 0;  // my outgoing payload (incl. self segment)
};

// pipe_chunk: relay ring chunk (reference staging geometry); direct_chunk:
// work-item size of direct pushes / pulls / self-ring chunks (<= pipe_chunk)
// and of local copies -- small enough that the last wave of items ends within
// a few microseconds across CTAs.
Schedule build_schedule(const PlanResult& plan, const RankBuffers& rb, uint64_t pipe_chunk, uint32_t slots,
                        uint64_t direct_chunk, uint64_t push_chunk = 0, uint64_t ll_max = 0);

// Item k of a flow, its key, and the host merge of the flows into the item
// list (`before` order) -- what the device generator reproduces.
Item cut_item(const CutDesc& f, uint64_t k);
double cut_key(const CutDesc& f, uint64_t k);
std::vector<Item> merge_cuts(const std::vector<CutDesc>& flows);
// Fill sc.items / sc.ll_items on the host from the cuts.
void materialize(Schedule& sc);

// Is pair (s, d), one end of which is me, built from several group
// operations?  (Never LL, never pulled or zero copy: pushed into the
// receiver's self ring and drained part by part.)
bool pair_is_multi(const RankBuffers& rb, int s, int d);

// Does pair (s, d) of `bytes` ride the LL protocol?  Both endpoints decide
// alike from what they both know: the pair size and the replicated plan
// (0 < bytes <= ll_max, no relay route).
bool ll_pair(const PlanResult& plan, int s, int d, uint64_t bytes, uint64_t ll_max);

// 1-GPU emulated exchange: every pair's segment as local copies (packed
// layout), as flows (merge_cuts gives the item list).
std::vector<CutDesc> build_local_cuts(int R, const uint64_t* matrix, const uint64_t* send_base,
                                      const uint64_t* recv_base, uint64_t chunk);

}  // namespace nb
