/* nimble.h -- C ABI of the B200-native NIMBLE data path.
 *
 * One shared library, paper_2604_00317_b200/libnimble_b200.so, exports every
 * symbol below.  No C++ or CUDA types cross this boundary: plain pointers,
 * sizes and opaque handles; streams are passed as `void*` (a cudaStream_t).
 * No call throws; every call returns a nimbleResult_t, and
 * nimbleGetLastError() returns the message of the last failure on the calling
 * thread.
 *
 * Three groups, each mirroring an existing interface:
 *
 *  1. Link-load model, traffic-matrix ingest and planner -- the reference's
 *     C++ planning API (/root/reference/proj/include/nimble/ headers), same
 *     semantics, bit-exact results; host-only, usable without a GPU.
 *  2. Communicator and data path -- shaped like NCCL 2.28.9's nccl.h (the
 *     interface the paper says NIMBLE sits behind): result
 *     codes nccl.h:42-50, data types nccl.h:300-313, unique id nccl.h:157,
 *     ncclCommInitRank nccl.h:171, ncclCommInitAll nccl.h:180,
 *     ncclCommDestroy nccl.h:192, ncclSend/ncclRecv nccl.h:507,526,
 *     ncclGroupStart/End nccl.h:558,568, ncclAlltoAll nccl.h:460-461,
 *     ncclCommRegister/Deregister, ncclMemAlloc/Free.
 *  3. Benchmark entry points mirroring the artifact's --p2p / --skewed runs
 *     (proj/tools/nimble.cpp:220-284) on real buffers.
 */
#ifndef NIMBLE_B200_H_
#define NIMBLE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NIMBLE_MAJOR 0
#define NIMBLE_MINOR 1
#define NIMBLE_PATCH 0
#define NIMBLE_VERSION_CODE (NIMBLE_MAJOR * 10000 + NIMBLE_MINOR * 100 + NIMBLE_PATCH)

/* Mirrors ncclResult_t (nccl.h:42-50). */
typedef enum {
    nimbleSuccess = 0,
    nimbleUnhandledCudaError = 1,
    nimbleSystemError = 2,
    nimbleInternalError = 3,
    nimbleInvalidArgument = 4,
    nimbleInvalidUsage = 5,
    nimbleRemoteError = 6,
    nimbleInProgress = 7,
    nimbleNumResults = 8
} nimbleResult_t;

/* Mirrors ncclDataType_t (nccl.h:300-313); only the element size matters. */
typedef enum {
    nimbleInt8 = 0, nimbleChar = 0,
    nimbleUint8 = 1,
    nimbleInt32 = 2, nimbleInt = 2,
    nimbleUint32 = 3,
    nimbleInt64 = 4,
    nimbleUint64 = 5,
    nimbleFloat16 = 6, nimbleHalf = 6,
    nimbleFloat32 = 7, nimbleFloat = 7,
    nimbleFloat64 = 8, nimbleDouble = 8,
    nimbleBfloat16 = 9,
    nimbleFloat8e4m3 = 10,
    nimbleFloat8e5m2 = 11,
    nimbleNumTypes = 12
} nimbleDataType_t;

const char* nimbleGetErrorString(nimbleResult_t result);
const char* nimbleGetLastError(void);
nimbleResult_t nimbleGetVersion(int* version);

/* ------------------------------------------------------------------ 1. planning */

/* proj/include/nimble/topology.hpp:36 (Fabric) */
typedef enum { nimbleFabricAllToAll = 0, nimbleFabricNvSwitch = 1 } nimbleFabric_t;
/* proj/include/nimble/topology.hpp:22 (LinkKind) */
typedef enum { nimbleLinkNvLink = 0, nimbleLinkSwitchPort = 1, nimbleLinkAttach = 2, nimbleLinkRail = 3 } nimbleLinkKind_t;
/* proj/include/nimble/planner.hpp:17 (PathClass) */
typedef enum { nimbleRouteDirect = 0, nimbleRouteTwoHop = 1, nimbleRouteRail = 2 } nimbleRoute_t;

typedef struct nimbleTopology* nimbleTopology_t;
typedef struct nimblePlan* nimblePlan_t;

/* replaces build_canonical (proj/include/nimble/topology.hpp:68-70, topology.cpp:119) */
nimbleResult_t nimbleTopologyCreate(int nodes, int gpus_per_node, int nics_per_node,
                                    double nvlink_bytes_per_s, double rail_bytes_per_s,
                                    nimbleFabric_t fabric, nimbleTopology_t* topo);
/* replaces load_topology / save_topology (topology.hpp:76-77) */
nimbleResult_t nimbleTopologyLoad(const char* text, nimbleTopology_t* topo);
nimbleResult_t nimbleTopologySave(nimbleTopology_t topo, char* out, size_t cap, size_t* need);
nimbleResult_t nimbleTopologyDestroy(nimbleTopology_t topo);
/* Topology::link_count / link(id) / link_name (topology.hpp:51-53) */
nimbleResult_t nimbleTopologyLinkCount(nimbleTopology_t topo, int* count);
nimbleResult_t nimbleTopologyLink(nimbleTopology_t topo, int id, int* kind, double* capacity,
                                  char* name, size_t name_cap);
/* per-link capacity override (the file format's "link <src> <dst> <gbps>") */
nimbleResult_t nimbleTopologySetCapacity(nimbleTopology_t topo, int id, double bytes_per_s);
/* Topology::port_up_id / port_down_id / nvlink_id (topology.hpp:57-59); -1 + error if absent */
nimbleResult_t nimbleTopologyLinkId(nimbleTopology_t topo, int kind, int node, int a, int b, int* id);

/* Traffic-matrix ingest: R*R row-major uint64 byte counts, row = sender.
 * replaces gen_p2p / gen_skewed_a2av / gen_stencil_1d / gen_aggregator /
 * gen_irregular (proj/include/nimble/workloads.hpp:39-56). */
nimbleResult_t nimbleGenP2P(int ranks, int src, int dst, uint64_t size, uint64_t* matrix);
nimbleResult_t nimbleGenSkewed(int ranks, uint64_t per_rank, double ratio, int hot_dst,
                               int per_sender_hot, uint64_t* matrix);
nimbleResult_t nimbleGenStencil1D(int ranks, uint64_t halo, uint64_t* matrix);
nimbleResult_t nimbleGenAggregator(int ranks, const int* dsts, int ndsts, uint64_t per_src,
                                   uint64_t* matrix);
nimbleResult_t nimbleGenIrregular(int ranks, uint64_t total, double sparsity, uint64_t seed,
                                  uint64_t* matrix);
/* write_payload_matrix / read_payload_matrix (workloads.hpp:58-59); `ranks`
 * in/out: capacity of `matrix` in entries on input, R on output. */
nimbleResult_t nimbleMatrixToText(int ranks, const uint64_t* matrix, char* out, size_t cap, size_t* need);
nimbleResult_t nimbleMatrixFromText(const char* text, uint64_t* matrix, size_t cap, int* ranks);

/* proj/include/nimble/planner.hpp:36-56 (CostModel + PlannerConfig) */
typedef struct {
    double lambda;                 /* 0.5 */
    uint64_t epsilon;              /* 4 MiB */
    double pi;                     /* 0.25 */
    uint64_t small_message_cutoff; /* 1 MiB */
    uint64_t saturation_intra;     /* 64 MiB */
    uint64_t saturation_inter;     /* 32 MiB */
    uint64_t max_pair_visits;      /* 1e6 */
    int normalize_by_capacity;     /* 1 */
} nimblePlannerConfig;

/* proj/include/nimble/planner.hpp:71-78 (PlanStats) */
typedef struct {
    uint64_t pair_visits, placements, fallback_pairs, residual_flows, refine_moves;
    double wall_seconds;
} nimblePlanStats;

nimbleResult_t nimblePlannerConfigDefault(nimblePlannerConfig* cfg);
/* replaces plan() (planner.hpp:99-100); ranks_per_node = RankMap block size */
nimbleResult_t nimblePlanCreate(nimbleTopology_t topo, int ranks, int ranks_per_node,
                                const uint64_t* matrix, const nimblePlannerConfig* cfg,
                                nimblePlan_t* plan);
/* replaces plan_direct_baseline() (planner.hpp:103-104) */
nimbleResult_t nimblePlanDirect(nimbleTopology_t topo, int ranks, int ranks_per_node,
                                const uint64_t* matrix, nimblePlan_t* plan);
/* replaces enumerate_paths() (planner.hpp:86-87): a plan handle holding one
 * pair (src, dst) with zero demand and no flows, whose candidates are the
 * enumerated routes (read them with nimblePlanCandidate). */
nimbleResult_t nimbleEnumeratePaths(nimbleTopology_t topo, int ranks, int ranks_per_node, int src, int dst,
                                    nimblePlan_t* paths);
nimbleResult_t nimblePlanDestroy(nimblePlan_t plan);
nimbleResult_t nimblePlanNumPairs(nimblePlan_t plan, int* npairs);
nimbleResult_t nimblePlanPair(nimblePlan_t plan, int pair, int* src, int* dst, uint64_t* demand,
                              int* ncandidates, int* nflows);
/* enumerate_paths() output for the pair (planner.hpp:19-30,86-87) */
nimbleResult_t nimblePlanCandidate(nimblePlan_t plan, int pair, int cand, int* route, int* via,
                                   int* rail, int* hops, int* edges, int edges_cap, int* nedges);
/* FlowAssignment (planner.hpp:58-61): the chunk-to-path assignment */
nimbleResult_t nimblePlanFlow(nimblePlan_t plan, int pair, int flow, int* cand, double* bytes);
nimbleResult_t nimblePlanGetStats(nimblePlan_t plan, nimblePlanStats* stats);
/* plan_link_loads / max_normalized_load (planner.hpp:106-107) */
nimbleResult_t nimblePlanLinkLoads(nimblePlan_t plan, double* loads, int nlinks);
nimbleResult_t nimblePlanMaxNormalizedLoad(nimblePlan_t plan, double* seconds);
/* plan_to_json (planner.hpp:109) */
nimbleResult_t nimblePlanToJson(nimblePlan_t plan, char* out, size_t cap, size_t* need);
/* plan_from_json (planner.hpp:110): re-enumerates routes on `topo`, matches
 * flows by (class, via, rail), checks every pair's flows sum to its demand. */
nimbleResult_t nimblePlanFromJson(nimbleTopology_t topo, int ranks, int ranks_per_node, const char* json,
                                  nimblePlan_t* plan);

/* ------------------------------------------------------------ 2. communicator */

#define NIMBLE_UNIQUE_ID_BYTES 128
typedef struct { char internal[NIMBLE_UNIQUE_ID_BYTES]; } nimbleUniqueId;
typedef struct nimbleComm* nimbleComm_t;

/* Runtime knobs of a communicator.  The planner runs on the comm's own
 * link-load model: by default the B200 box as it is (nvswitch, 900 GB/s per
 * port), which plans every pair direct; fabric = nimbleFabricAllToAll with
 * gpus_per_node > nranks exercises the reference's mesh model, whose relay
 * routes the forwarding engine then executes through peer staging rings. */
typedef struct {
    nimbleFabric_t fabric;        /* link-load model the planner charges     */
    int gpus_per_node;            /* model GPUs (>= nranks); idle ones relay */
    double nvlink_bytes_per_s;    /* per link / port                          */
    nimblePlannerConfig planner;
    uint64_t pipe_chunk;          /* relay staging slot size, 64 KiB (reference: 512 KiB,
                                     pipeline.hpp:19; finer slots keep more CTAs busy)  */
    uint64_t p2p_buffer;          /* staging bytes per ring, 10 MiB (pipeline.hpp:18);
                                     slots = channels * p2p_buffer / pipe_chunk <= 256  */
    int channels_per_peer;        /* rings per relayed flow, 1 (pipeline.hpp:23)        */
    int ctas;                     /* forwarding-engine CTAs per launch, 0 = auto        */
    uint64_t direct_chunk;        /* work-item size of direct pulls and local copies
                                     (<= pipe_chunk), 0 = auto (128 KiB, capped at
                                     pipe_chunk = 64 KiB)                                  */
    int pull;                     /* receiver-driven pulls.  0 = auto (default): receivers
                                     ask; a registered sender grants unless its own port is
                                     ingress-bound (ingress > 1.2 x egress; 1.55 x with two
                                     ranks), in which case it pushes out; 1 = never (push
                                     only); 2 = always grant                             */
    uint64_t push_chunk;          /* work-item size of direct pushes and of the staged self
                                     rings that mirror them (<= pipe_chunk), 0 = auto
                                     (8 KiB).  A port that pulls in while it pushes out runs
                                     both through one CTA ring; short pushes keep a store
                                     stalled on a busy egress from holding up the pulls   */
    uint64_t ll_max;              /* direct pairs of at most ll_max bytes (<= 1 MiB) take the
                                     low-latency protocol: the sender stores data with the
                                     epoch flag inline into the receiver's LL slot, and no
                                     posts, fences or completion handshake are needed.
                                     Default 1 MiB; 0 disables                           */
} nimbleCommConfig;

nimbleResult_t nimbleCommConfigDefault(nimbleCommConfig* cfg);

nimbleResult_t nimbleGetUniqueId(nimbleUniqueId* uniqueId);
/* One process per GPU (uses the calling thread's current CUDA device). */
nimbleResult_t nimbleCommInitRank(nimbleComm_t* comm, int nranks, nimbleUniqueId commId, int rank);
/* One process, `ndev` GPUs (devlist NULL = 0..ndev-1). */
nimbleResult_t nimbleCommInitAll(nimbleComm_t* comms, int ndev, const int* devlist);
nimbleResult_t nimbleCommDestroy(nimbleComm_t comm);
nimbleResult_t nimbleCommCount(const nimbleComm_t comm, int* count);
nimbleResult_t nimbleCommUserRank(const nimbleComm_t comm, int* rank);
nimbleResult_t nimbleCommCuDevice(const nimbleComm_t comm, int* device);
/* Device-side failures (flag-wait timeout, size mismatch) surface here. */
nimbleResult_t nimbleCommGetAsyncError(nimbleComm_t comm, nimbleResult_t* asyncError);
/* Collective across the comm; every rank must pass an equal config. */
nimbleResult_t nimbleCommSetConfig(nimbleComm_t comm, const nimbleCommConfig* cfg);
nimbleResult_t nimbleCommGetConfig(nimbleComm_t comm, nimbleCommConfig* cfg);

/* Buffer registration (ncclCommRegister/Deregister).  Collective: every rank
 * registers one buffer per call, in the same order.  Receive buffers inside a
 * registered window are written in place by peers (zero copy); unregistered
 * receive buffers are fed through the comm's staging rings. */
nimbleResult_t nimbleCommRegister(const nimbleComm_t comm, void* buff, size_t size, void** handle);
nimbleResult_t nimbleCommDeregister(const nimbleComm_t comm, void* handle);
nimbleResult_t nimbleMemAlloc(void** ptr, size_t size);
nimbleResult_t nimbleMemFree(void* ptr);

/* Group semantics follow NCCL: ops are enqueued and one exchange per comm is
 * launched at GroupEnd.  Several sends to (receives from) one peer in a group
 * are matched in issue order with the peer's receives (sends), each pair of
 * matching operations having the same byte count (ncclSend / ncclRecv
 * rules); such a pair is pushed through the receiver's staging ring and
 * drained into each receive buffer in turn (nvswitch model only). */
nimbleResult_t nimbleGroupStart(void);
nimbleResult_t nimbleGroupEnd(void);
nimbleResult_t nimbleSend(const void* sendbuff, size_t count, nimbleDataType_t datatype, int peer,
                          nimbleComm_t comm, void* stream);
nimbleResult_t nimbleRecv(void* recvbuff, size_t count, nimbleDataType_t datatype, int peer,
                          nimbleComm_t comm, void* stream);
nimbleResult_t nimbleAlltoAll(const void* sendbuff, void* recvbuff, size_t count,
                              nimbleDataType_t datatype, nimbleComm_t comm, void* stream);
/* counts / displacements in elements of `datatype`, as MPI_Alltoallv.
 * Stream semantics as NCCL's: the exchange is ordered after earlier work on
 * `stream` and later work waits for it.  Back-to-back exchanges of one comm on
 * one stream overlap the previous one's completion (its next launch chains on
 * the previous exchange's epoch on the device, ~5 us less per call); work
 * enqueued between two exchanges is always waited for (NIMBLE_CHAIN=0
 * disables the chaining). */
nimbleResult_t nimbleAlltoAllv(const void* sendbuff, const size_t sendcounts[], const size_t sdispls[],
                               void* recvbuff, const size_t recvcounts[], const size_t rdispls[],
                               nimbleDataType_t datatype, nimbleComm_t comm, void* stream);

/* Single-GPU emulation of an R-rank exchange: one kernel moves every pair's
 * segment (packed MPI layout) between R send and R receive buffers on the
 * current device -- the 1-GPU local-copy calibration of the forwarding engine. */
nimbleResult_t nimbleExchangeLocal(int ranks, const void* const* sendbuffs, void* const* recvbuffs,
                                   const uint64_t* matrix, int ctas, void* stream);

/* Payload helpers (device): byte j of pair (s,d) is byte j%8 of
 * splitmix64(seed ^ s<<48 ^ d<<40 ^ j/8).  Check adds mismatching bytes into
 * *mismatches (device pointer, uint64). */
nimbleResult_t nimbleFillPayload(void* buf, uint64_t first, uint64_t nbytes, uint64_t seed, int src,
                                 int dst, void* stream);
nimbleResult_t nimbleCheckPayload(const void* buf, uint64_t first, uint64_t nbytes, uint64_t seed,
                                  int src, int dst, uint64_t* mismatches, void* stream);

/* --------------------------------------------------------- 3. bench entry points */

typedef struct {
    double seconds_median;   /* per exchange, max over ranks, CUDA events     */
    double seconds_min;
    double gbps_effective;   /* total payload bytes / seconds_median / 1e9    */
    double bound_seconds;    /* MCF port bound of the matrix on this box      */
    double plan_seconds;     /* host planner wall time for this matrix        */
    uint64_t total_bytes;
    uint64_t mismatches;     /* delivered bytes that differ from the payload  */
    int relay_flows;         /* flows the plan routes through a relay          */
} nimbleBenchResult;

/* --p2p: `bytes` from src to dst (collective over the comm). */
nimbleResult_t nimbleBenchP2P(nimbleComm_t comm, uint64_t bytes, int src, int dst, int warmup,
                              int iters, nimbleBenchResult* result);
/* --skewed: gen_skewed_a2av(nranks, per_rank, ratio, hot) (collective). */
nimbleResult_t nimbleBenchSkewed(nimbleComm_t comm, uint64_t per_rank, double ratio, int hot,
                                 int warmup, int iters, nimbleBenchResult* result);
/* Any R*R matrix (packed layout), e.g. gen_irregular output (collective). */
nimbleResult_t nimbleBenchMatrix(nimbleComm_t comm, const uint64_t* matrix, int warmup, int iters,
                                 nimbleBenchResult* result);

/* ------------------------------------------------------------- diagnostics */

/* Host-only: join the out-of-band rendezvous of `id` as (rank, nranks), all-
 * gather `n` bytes per rank into `out` (nranks * n bytes, rank order), leave.
 * Exercises the bootstrap that nimbleCommInitRank uses, without a GPU. */
nimbleResult_t nimbleBootstrapAllgather(const nimbleUniqueId* id, int rank, int nranks, const void* in, size_t n,
                                        void* out);

/* Host-only: the host shared-memory allgather communicators use for per-call
 * metadata (the mesh model's demand rows), `rounds` times back to back; every
 * round checks that each record is that round's, from its rank.  `out` gets
 * the last round's records (nranks * n bytes, n <= 248). */
nimbleResult_t nimbleBootstrapShmAllgather(const nimbleUniqueId* id, int rank, int nranks, const void* in, size_t n,
                                           void* out, int rounds);

/* The chunk scheduler, host only: the ordered work items rank `rank` would
 * run for `plan` (from nimblePlanCreate / nimblePlanDirect over `ranks` ranks,
 * packed layout).  recv_staged_mask bit s: my receive segment from s is not
 * registered (drained through my self ring); pull_mask bit s: I ask s to let
 * me pull.  Items are written as nimbleItem records in execution order;
 * addresses are synthetic: send segment for d at (1 + rank) << 40 + sdispl[d],
 * receive segment from s at (17 + rank) << 40 + rdispl[s]. */
typedef struct {
    uint64_t src, dst;  /* absolute (local kinds) or offset inside the pair segment */
    uint32_t bytes;
    uint8_t kind;       /* 0 local, 1 push, 2 stage, 3 forward, 4 pull */
    uint8_t peer;       /* receiver (push/forward), relay (stage), sender (pull) */
    uint16_t aux;       /* final receiver (stage), original sender (forward) */
    uint32_t seq;       /* chunk index inside its ring / flow */
    uint32_t pad;
} nimbleItem;
nimbleResult_t nimbleDebugSchedule(nimblePlan_t plan, int rank, int ranks, uint64_t pipe_chunk, uint32_t slots,
                                   uint64_t direct_chunk, uint64_t push_chunk, uint64_t recv_staged_mask,
                                   uint64_t pull_mask,
                                   nimbleItem* items, int cap, int* nitems);

/* The same item list produced by the device-side generator (engine.cu,
 * gen_items_kernel) on the current CUDA device: the flows go to the GPU as
 * kernel parameters and are merged there -- how a communicator schedules a
 * new matrix without a host merge or an upload.  Must equal
 * nimbleDebugSchedule's list item for item. */
nimbleResult_t nimbleDebugScheduleDevice(nimblePlan_t plan, int rank, int ranks, uint64_t pipe_chunk,
                                         uint32_t slots, uint64_t direct_chunk, uint64_t push_chunk,
                                         uint64_t recv_staged_mask, uint64_t pull_mask,
                                         nimbleItem* items, int cap, int* nitems);

/* Device timeline of the comm's last launch (%globaltimer ns): kernel start,
 * prologue done, first item, last item, CTAs done, completions signalled,
 * completions observed, first CTA done, latest work loops done, latest
 * completion fence, earliest work loops done (16 slots); then, for CTA i < 160,
 * 6 words at 16 + 6 i: first item, queue empty, loops done, fence done (ns),
 * bytes stored into peers, bytes pulled or copied locally.  Needs
 * NIMBLE_TRACE=1 at comm creation; n >= 16 (up to 976 words are written). */
nimbleResult_t nimbleCommDebugTrace(nimbleComm_t comm, uint64_t* out, int n);

/* Device counters of the forwarding engine, accumulated over the comm's
 * launches (NIMBLE_STATS=1 at comm creation, on every rank).  bytes/items are
 * indexed [kind][peer]: kind 0 local copy, 1 push (by receiver), 2 stage into
 * a relay's ring (by relay), 3 forward out of a ring hosted here (by final
 * receiver), 4 pull (by sender), 5 LL send (by receiver), 6 LL receive (by
 * sender), 7 drain of my own staged-receive ring (by sender).  The slot
 * counters check the bounded-buffer invariant of the staging rings on the
 * device (proj/tests/acceptance.cpp:270-288, occupancy <= S): the largest
 * number of claimed-not-drained slots any of my stager claims observed in its
 * ring, and the number of claims of a slot whose previous chunk had not been
 * drained (must be 0).  reset != 0 zeroes the counters after reading. */
typedef struct {
    uint64_t bytes[8][32];
    uint64_t items[8][32];
    uint64_t slot_max_occupancy;
    uint64_t slot_double_claims;
    uint64_t slot_claims;
    uint64_t pad;
    /* host side: the C ABI's cost per data-path call (nimbleAlltoAllv /
     * grouped send-recv), and the plans / schedules built for new matrices */
    uint64_t host_calls, host_ns, host_ns_max;
    uint64_t plans_built, plan_ns, schedules_built, schedule_ns;
    uint64_t host_pad;
} nimbleCommStats;
nimbleResult_t nimbleCommGetStats(nimbleComm_t comm, nimbleCommStats* stats, int reset);

#ifdef __cplusplus
}
#endif

#endif /* NIMBLE_B200_H_ */
