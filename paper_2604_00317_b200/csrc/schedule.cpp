// Chunk scheduler; see schedule.hpp.
#include "schedule.hpp"

#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "capi_util.hpp"

namespace nb {

namespace {

struct Cuts {
    std::vector<CutDesc> flows;
    uint32_t count = 0;  // items so far
};

// Appends one flow (device.cuh CutDesc); returns its item count.
uint32_t cut(Cuts& out, Item proto, uint64_t src0, uint64_t dst0, uint64_t bytes, uint64_t chunk, double phase,
             bool pull = false, uint64_t src_from_dst = 0, double scale = 1.0) {
    const uint64_t n = (bytes + chunk - 1) / chunk;
    if (n) {
        CutDesc c{};
        c.proto = proto;
        c.src0 = src0;
        c.dst0 = dst0;
        c.bytes = bytes;
        c.chunk = chunk;
        c.n = n;
        c.src_from_dst = src_from_dst;
        c.phase = phase;
        c.scale = scale;
        c.base = out.count;
        c.flags = (src0 ? static_cast<uint32_t>(kCutSrc) : 0u) | kCutDst | (pull ? static_cast<uint32_t>(kCutPull) : 0u);
        out.flows.push_back(c);
    }
    out.count += static_cast<uint32_t>(n);
    return static_cast<uint32_t>(n);
}

struct Cursor {
    double key;
    const CutDesc* f;
    uint64_t k;
};

// Strict, total order: key, then hot (larger) flows first on ties, then insertion order.
bool before(const Cursor& a, const Cursor& b) {
    if (a.key != b.key) return a.key < b.key;
    if (a.f->bytes != b.f->bytes) return a.f->bytes > b.f->bytes;
    return a.f->base + a.k < b.f->base + b.k;
}

}  // namespace

Item cut_item(const CutDesc& f, uint64_t k) {
    Item it = f.proto;
    const uint64_t off = k * f.chunk;
    it.src = (f.flags & kCutSrc) ? f.src0 + off : 0;
    it.dst = (f.flags & kCutDst) ? f.dst0 + off : 0;
    it.bytes = static_cast<uint32_t>(std::min(f.chunk, f.bytes - off));
    it.seq = f.proto.seq + static_cast<uint32_t>(k);
    if (f.flags & kCutPull) it.src = it.dst - f.src_from_dst;
    return it;
}

double cut_key(const CutDesc& f, uint64_t k) {
    return (static_cast<double>(k) + 0.5) / static_cast<double>(f.n) * f.scale + f.phase;
}

// All items in `before` order: a k-way merge over the flows (each one's keys
// increase with k), generating items as they are emitted -- O(n log flows)
// with no per-item sort records.
std::vector<Item> merge_cuts(const std::vector<CutDesc>& flows) {
    std::vector<Cursor> heap;
    heap.reserve(flows.size());
    uint64_t total = 0;
    for (const CutDesc& f : flows) {
        heap.push_back({cut_key(f, 0), &f, 0});
        total += f.n;
    }
    auto later = [](const Cursor& a, const Cursor& b) { return before(b, a); };  // min-heap
    std::make_heap(heap.begin(), heap.end(), later);
    std::vector<Item> items;
    items.reserve(total);
    while (!heap.empty()) {
        std::pop_heap(heap.begin(), heap.end(), later);
        Cursor& c = heap.back();
        items.push_back(cut_item(*c.f, c.k));
        if (++c.k == c.f->n) {
            heap.pop_back();
        } else {
            c.key = cut_key(*c.f, c.k);
            std::push_heap(heap.begin(), heap.end(), later);
        }
    }
    return items;
}

void materialize(Schedule& sc) {
    sc.items = merge_cuts(sc.cuts);
    if (sc.n_push_lane) {  // the push lane first, each queue in merge order (what the generator writes)
        std::vector<CutDesc> lane, main;
        for (const CutDesc& f : sc.cuts) ((f.flags & kCutPushLane) ? lane : main).push_back(f);
        std::vector<Item> a = merge_cuts(lane), b = merge_cuts(main);
        a.insert(a.end(), b.begin(), b.end());
        sc.items = std::move(a);
    }
    sc.ll_items.clear();
    for (const CutDesc& f : sc.ll_cuts)
        for (uint64_t k = 0; k < f.n; ++k) sc.ll_items.push_back(cut_item(f, k));
}

namespace {

constexpr double kHop2 = 1e-9;  // forward of chunk k sorts right after its stage-in

// A pair made of several group operations (NCCL: several sends to, or
// receives from, one peer in a group, matched in order).
bool multi(const std::vector<std::vector<std::pair<uint64_t, uint64_t>>>& parts, int peer) {
    return static_cast<size_t>(peer) < parts.size() && parts[static_cast<size_t>(peer)].size() > 1;
}

// Each part (ptr, offset inside the pair, bytes, first chunk index).
template <typename F>
void each_part(const std::vector<std::pair<uint64_t, uint64_t>>& parts, uint64_t chunk, F&& f) {
    uint64_t off = 0;
    uint32_t seq = 0;
    for (const auto& [ptr, bytes] : parts) {
        f(ptr, off, bytes, seq);
        off += bytes;
        seq += static_cast<uint32_t>((bytes + chunk - 1) / chunk);
    }
}

// Experiment knobs (environment, read once; identical on every rank):
//  NIMBLE_PUSH_SPAN = a in (0, 1]: direct pushes (and the self-ring drains
//    that mirror them) take keys in [0, a): a port that pushes out while it
//    pulls in finishes its stores -- and their acknowledgements, which its
//    completion fence waits for -- before its pulls end;
//  NIMBLE_PULL_TAIL = bytes: the last bytes of every pull flow are cut into
//    NIMBLE_PULL_TAIL_CHUNK pieces, so the CTAs run out of work together.
struct Knobs {
    double push_span = 1.0;
    uint64_t pull_tail = 0, pull_tail_chunk = 16 << 10;
    Knobs() {
        if (const char* e = std::getenv("NIMBLE_PUSH_SPAN"); e && *e) push_span = std::strtod(e, nullptr);
        if (!(push_span > 0.0 && push_span <= 1.0)) push_span = 1.0;
        if (const char* e = std::getenv("NIMBLE_PULL_TAIL"); e && *e) pull_tail = std::strtoull(e, nullptr, 0);
        if (const char* e = std::getenv("NIMBLE_PULL_TAIL_CHUNK"); e && *e)
            pull_tail_chunk = std::max<uint64_t>(4096, std::strtoull(e, nullptr, 0));
    }
};

const Knobs& knobs() {
    static const Knobs k;
    return k;
}

// part keys span [off / total, (off + bytes) / total): the pair's progress
double part_phase(uint64_t off, uint64_t total) { return static_cast<double>(off) / static_cast<double>(total); }
double part_scale(uint64_t bytes, uint64_t total) { return static_cast<double>(bytes) / static_cast<double>(total); }

}  // namespace

bool pair_is_multi(const RankBuffers& rb, int s, int d) {
    return s == rb.me ? multi(rb.send_parts, d) : d == rb.me ? multi(rb.recv_parts, s) : false;
}

bool ll_pair(const PlanResult& plan, int s, int d, uint64_t bytes, uint64_t ll_max) {
    if (s == d || bytes == 0 || bytes > ll_max || bytes > kLLMaxData) return false;
    for (const PairRoutes& pr : plan.pairs)
        if (pr.src == s && pr.dst == d) {
            for (const Flow& f : pr.flows)
                if (pr.cands[static_cast<size_t>(f.cand)].route != Route::Direct) return false;
            return true;
        }
    return true;  // not in the plan: a direct pair
}

Schedule build_schedule(const PlanResult& plan, const RankBuffers& rb, uint64_t pipe_chunk, uint32_t slots,
                        uint64_t direct_chunk, uint64_t push_chunk, uint64_t ll_max) {
    const int R = rb.R, me = rb.me;
    if (R > kMaxRanks) throw Error(nimbleInvalidArgument, "schedule: too many ranks");
    if (pipe_chunk == 0 || pipe_chunk > 0xffffffffull) throw Error(nimbleInvalidArgument, "schedule: bad pipe_chunk");
    if (slots == 0 || slots > kMaxSlots) throw Error(nimbleInvalidArgument, "schedule: bad slot count");
    const uint64_t dchunk = std::min<uint64_t>(std::max<uint64_t>(direct_chunk, 4096), pipe_chunk);
    const uint64_t schunk = push_chunk ? std::min<uint64_t>(std::max<uint64_t>(push_chunk, 4096), pipe_chunk) : dchunk;
    Schedule sc;
    const double span = knobs().push_span;
    sc.posts = rb.recv_post;
    sc.send_posts = rb.send_post;
    Cuts keyed;

    // self segment: local copy
    if (rb.send_bytes[me] != rb.recv_bytes[me])
        throw Error(nimbleInvalidArgument, "alltoallv: self send and receive counts differ");
    if (rb.send_bytes[me]) {
        Item proto{};
        proto.kind = kLocal;
        proto.peer = static_cast<uint8_t>(me);
        cut(keyed, proto, rb.send_ptr[me], rb.recv_ptr[me], rb.send_bytes[me], dchunk, 0.0);
        sc.moved_bytes += rb.send_bytes[me];
    }

    Cuts ll_send, ll_recv;
    for (const PairRoutes& pr : plan.pairs) {
        const int s = pr.src, d = pr.dst;
        if ((s == me || d == me) && !pair_is_multi(rb, s, d) && ll_pair(plan, s, d, pr.demand, ll_max)) {
            if (s == me && pr.demand != rb.send_bytes[d])
                throw Error(nimbleInvalidArgument, "schedule: plan demand differs from the send count");
            if (d == me && pr.demand != rb.recv_bytes[s])
                throw Error(nimbleInvalidArgument, "alltoallv: receive count differs from the planned demand");
            // pieces of kLLPiece bytes: several CTAs per pair; the pair size rides in pad
            Item proto{};
            proto.pad = static_cast<uint32_t>(pr.demand);
            if (s == me) {
                proto.kind = kLLSend;
                proto.peer = static_cast<uint8_t>(d);
                cut(ll_send, proto, rb.send_ptr[d], 0, pr.demand, kLLPiece, 0.0);
                ll_send.flows.back().flags = kCutSrc;  // no destination address: the receiver's LL slot
                sc.moved_bytes += pr.demand;
            } else {
                proto.kind = kLLRecv;
                proto.peer = static_cast<uint8_t>(s);
                cut(ll_recv, proto, 0, rb.recv_ptr[s], pr.demand, kLLPiece, 0.0);
                sc.ll_senders |= 1ull << s;
            }
            continue;
        }
        if (s != me && d != me) {
            // only relay duty can involve me
            bool relays_me = false;
            for (const Flow& f : pr.flows)
                relays_me |= pr.cands[static_cast<size_t>(f.cand)].via == me;
            if (!relays_me) continue;
        }
        if (s == me && pr.demand != rb.send_bytes[d])
            throw Error(nimbleInvalidArgument, "schedule: plan demand differs from the send count");
        if (d == me && pr.demand != rb.recv_bytes[s])
            throw Error(nimbleInvalidArgument, "alltoallv: receive count differs from the planned demand");
        uint64_t off = 0;
        for (const Flow& f : pr.flows) {
            const Candidate& c = pr.cands[static_cast<size_t>(f.cand)];
            const uint64_t bytes = static_cast<uint64_t>(f.bytes);
            if (static_cast<double>(bytes) != f.bytes) throw Error(nimbleInternalError, "schedule: fractional flow");
            if (c.route == Route::Rail) throw Error(nimbleInvalidUsage, "schedule: inter-node rail routes need a multi-node box");
            if (c.route == Route::Direct) {
                if (s == me && multi(rb.send_parts, d)) {
                    // several sends to d in one group: one cut per part, chunk
                    // indices and progress keys continuing across the parts
                    // (the receiver cuts its receives identically)
                    if (bytes != pr.demand) throw Error(nimbleInvalidUsage, "group: several sends to one peer need a direct route");
                    Item proto{};
                    proto.kind = kPush;
                    proto.peer = static_cast<uint8_t>(d);
                    each_part(rb.send_parts[d], schunk, [&](uint64_t ptr, uint64_t po, uint64_t pb, uint32_t seq0) {
                        proto.seq = seq0;
                        sc.push_items[d] += cut(keyed, proto, ptr, po, pb, schunk, span * part_phase(po, pr.demand), false,
                                                0, span * part_scale(pb, pr.demand));
                    });
                    sc.push_targets |= 1ull << d;
                    sc.write_targets |= 1ull << d;
                    sc.moved_bytes += bytes;
                } else if (s == me) {
                    Item proto{};
                    proto.kind = kPush;
                    proto.peer = static_cast<uint8_t>(d);
                    sc.push_items[d] += cut(keyed, proto, rb.send_ptr[d] + off, off, bytes, schunk, 0.0, false, 0, span);
                    sc.push_targets |= 1ull << d;
                    sc.write_targets |= 1ull << d;
                    sc.moved_bytes += bytes;
                }
                if (d == me && multi(rb.recv_parts, s)) {
                    // several receives from s: staged through my self ring,
                    // each part drained to its own buffer (absolute addresses)
                    if (bytes != pr.demand) throw Error(nimbleInvalidUsage, "group: several receives from one peer need a direct route");
                    sc.recv_direct |= 1ull << s;
                    Item proto{};
                    proto.kind = kForward;
                    proto.peer = static_cast<uint8_t>(me);
                    proto.aux = static_cast<uint16_t>(s);
                    each_part(rb.recv_parts[s], schunk, [&](uint64_t ptr, uint64_t po, uint64_t pb, uint32_t seq0) {
                        proto.seq = seq0;
                        cut(keyed, proto, 0, ptr, pb, schunk, span * part_phase(po, pr.demand) + kHop2, false, 0,
                            span * part_scale(pb, pr.demand));
                    });
                } else if (d == me) {
                    sc.recv_direct |= 1ull << s;
                    if (rb.recv_post[s].mode & kPostPullRequest) {  // used if the sender grants it at run time
                        sc.pull_req |= 1ull << s;
                        Item proto{};
                        proto.kind = kPull;
                        proto.peer = static_cast<uint8_t>(s);
                        // source: offset inside the sender's segment
                        const uint64_t tail = knobs().pull_tail < bytes ? knobs().pull_tail : 0;
                        if (tail) {  // body at dchunk, the last `tail` bytes finer (same progress keys overall)
                            const uint64_t body = bytes - tail;
                            sc.pull_items[s] += cut(keyed, proto, 0, rb.recv_ptr[s] + off, body, dchunk, 0.0, true,
                                                  rb.recv_ptr[s], part_scale(body, bytes));
                            sc.pull_items[s] += cut(keyed, proto, 0, rb.recv_ptr[s] + off + body, tail,
                                                  knobs().pull_tail_chunk, part_phase(body, bytes), true, rb.recv_ptr[s],
                                                  part_scale(tail, bytes));
                        } else {
                            sc.pull_items[s] += cut(keyed, proto, 0, rb.recv_ptr[s] + off, bytes, dchunk, 0.0, true,
                                                  rb.recv_ptr[s]);
                        }
                    }
                    if ((rb.recv_post[s].mode & 0xf) == kPostStaged) {  // drain my self ring (s, me)
                        Item proto{};
                        proto.kind = kForward;
                        proto.peer = static_cast<uint8_t>(me);
                        proto.aux = static_cast<uint16_t>(s);
                        // chunk k of the ring is the sender's push item k: same cut
                        cut(keyed, proto, 0, off, bytes, schunk, kHop2, false, 0, span);
                    } else {
                        sc.recv_zc |= 1ull << s;
                    }
                }
            } else {  // two-hop relay through GPU `via`
                const int v = c.via;
                if (v < 0 || v >= R) throw Error(nimbleInvalidUsage, "schedule: relay GPU is not a rank of this comm");
                if (s == me) {
                    ++sc.relay_flows;
                    Item proto{};
                    proto.kind = kStage;
                    proto.peer = static_cast<uint8_t>(v);
                    proto.aux = static_cast<uint16_t>(d);
                    cut(keyed, proto, rb.send_ptr[d] + off, off, bytes, pipe_chunk, 0.0);
                    sc.moved_bytes += bytes;
                    // before returning, the last chunk of every used slot must be drained
                    const uint64_t n = (bytes + pipe_chunk - 1) / pipe_chunk;
                    for (uint64_t k = n > slots ? n - slots : 0; k < n; ++k) {
                        sc.final_waits.push_back(FlagLayout::consumed_off(R, d, v, static_cast<int>(k % slots)));
                        sc.final_waits.push_back(k);
                    }
                }
                if (v == me) {
                    Item proto{};
                    proto.kind = kForward;
                    proto.peer = static_cast<uint8_t>(d);
                    proto.aux = static_cast<uint16_t>(s);
                    sc.fwd_items[d] += cut(keyed, proto, 0, off, bytes, pipe_chunk, kHop2);
                    sc.write_targets |= 1ull << d;
                }
                if (d == me) sc.relay_writers |= 1ull << v;
            }
            off += bytes;
        }
    }
    sc.cuts = std::move(keyed.flows);
    sc.nitems = keyed.count;
    sc.n_ll_send = ll_send.count;
    sc.n_ll_recv = ll_recv.count;
    sc.ll_cuts = std::move(ll_send.flows);
    for (CutDesc& f : ll_recv.flows) f.base += ll_send.count;  // base = the piece's slot in ll_items
    sc.ll_cuts.insert(sc.ll_cuts.end(), ll_recv.flows.begin(), ll_recv.flows.end());
    return sc;
}

std::vector<CutDesc> build_local_cuts(int R, const uint64_t* m, const uint64_t* send_base, const uint64_t* recv_base,
                                      uint64_t chunk) {
    Cuts keyed;
    for (int s = 0; s < R; ++s) {
        uint64_t soff = 0;
        for (int d = 0; d < R; ++d) {
            const uint64_t b = m[static_cast<size_t>(s) * R + d];
            if (b) {
                uint64_t roff = 0;
                for (int x = 0; x < s; ++x) roff += m[static_cast<size_t>(x) * R + d];
                Item proto{};
                proto.kind = kLocal;
                proto.peer = static_cast<uint8_t>(d);
                cut(keyed, proto, send_base[s] + soff, recv_base[d] + roff, b, chunk, 0.0);
            }
            soff += b;
        }
    }
    return std::move(keyed.flows);
}

}  // namespace nb
