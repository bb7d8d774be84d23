/* TEST INFRASTRUCTURE ONLY -- the checker and the CPU data-movement baseline.
 *
 * The reference moves no bytes: its "CPU path" ends at a
 * plan plus a modelled completion time (proj/src/planner.cpp:320-429,
 * proj/src/simulator.cpp:226-262).  Delivery parity is therefore pinned by this
 * plain-C restatement of all-to-allv semantics over seeded payload bytes
 * ("Delivered receive buffers"):
 *
 *     recv_d[rdispl_d[s] .. + D[s][d]] == send_s[sdispl_s[d] .. + D[s][d]]
 *
 * with the packed (MPI_Alltoallv) layout sdispl_s[d] = sum_{d'<d} D[s][d'] and
 * rdispl_d[s] = sum_{s'<s} D[s'][d], and payload byte j of pair (s,d) equal to
 * byte (j % 8) (little endian) of splitmix64(seed ^ s<<48 ^ d<<40 ^ j/8)
 * (SURVEY.md sec. 8(d)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t pair_key(uint64_t seed, int s, int d) {
    return seed ^ ((uint64_t)s << 48) ^ ((uint64_t)d << 40);
}

/* Payload of pair (s,d), bytes [first, first+n) of the segment. */
void orc_fill(uint8_t* out, uint64_t first, uint64_t n, uint64_t seed, int s, int d) {
    uint64_t key = pair_key(seed, s, d);
    for (uint64_t j = 0; j < n; ++j) {
        uint64_t b = first + j;
        out[j] = (uint8_t)(splitmix64(key ^ (b >> 3)) >> (8 * (b & 7)));
    }
}

/* Number of bytes in [p, p+n) that differ from the payload of (s,d) at offset first. */
uint64_t orc_check(const uint8_t* p, uint64_t first, uint64_t n, uint64_t seed, int s, int d) {
    uint64_t key = pair_key(seed, s, d), bad = 0;
    for (uint64_t j = 0; j < n; ++j) {
        uint64_t b = first + j;
        bad += p[j] != (uint8_t)(splitmix64(key ^ (b >> 3)) >> (8 * (b & 7)));
    }
    return bad;
}

/* Packed displacements: sdispl[s*R+d] and rdispl[d*R+s]. */
void orc_displs(int R, const uint64_t* m, uint64_t* sdispl, uint64_t* rdispl) {
    for (int s = 0; s < R; ++s) {
        uint64_t acc = 0;
        for (int d = 0; d < R; ++d) {
            sdispl[s * R + d] = acc;
            acc += m[s * R + d];
        }
    }
    for (int d = 0; d < R; ++d) {
        uint64_t acc = 0;
        for (int s = 0; s < R; ++s) {
            rdispl[d * R + s] = acc;
            acc += m[s * R + d];
        }
    }
}

/* Reference delivery: recv_d <- send_s for every pair, single thread. */
void orc_alltoallv(int R, const uint64_t* m, uint8_t* const* send, uint8_t* const* recv) {
    uint64_t* sd = malloc(sizeof(uint64_t) * R * R);
    uint64_t* rd = malloc(sizeof(uint64_t) * R * R);
    orc_displs(R, m, sd, rd);
    for (int s = 0; s < R; ++s)
        for (int d = 0; d < R; ++d)
            if (m[s * R + d]) memcpy(recv[d] + rd[d * R + s], send[s] + sd[s * R + d], m[s * R + d]);
    free(sd);
    free(rd);
}

/* ---- multi-threaded CPU exchange (the timed CPU baseline) ---- */

typedef struct {
    const uint8_t* src;
    uint8_t* dst;
    uint64_t n;
} orc_piece;

typedef struct {
    orc_piece* pieces;
    int npieces;
    int tid, nthreads;
} orc_job;

static void* orc_worker(void* arg) {
    orc_job* j = (orc_job*)arg;
    for (int i = j->tid; i < j->npieces; i += j->nthreads)
        memcpy(j->pieces[i].dst, j->pieces[i].src, j->pieces[i].n);
    return NULL;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* Every flow (s, d, via, bytes) moves a contiguous range of the pair segment, in
 * flow order (direct first, then relays in candidate order); a relayed range is
 * copied twice (src -> staging[via] -> dst), as the store-and-forward pipeline
 * does.  Pieces are cut at `piece` bytes and spread round-robin over threads.
 * Returns wall seconds of the copy phase. */
double orc_exchange_flows(int R, const uint64_t* m, uint8_t* const* send, uint8_t* const* recv,
                          int nflows, const int* fsrc, const int* fdst, const int* fvia,
                          const double* fbytes, uint8_t* const* staging, uint64_t piece,
                          int nthreads) {
    uint64_t* sd = malloc(sizeof(uint64_t) * R * R);
    uint64_t* rd = malloc(sizeof(uint64_t) * R * R);
    uint64_t* pair_done = calloc((size_t)R * R, sizeof(uint64_t));
    uint64_t* stage_off = calloc((size_t)R, sizeof(uint64_t));
    orc_displs(R, m, sd, rd);
    if (piece == 0) piece = 1 << 20;
    size_t cap = 1024, n1 = 0, n2 = 0;
    orc_piece* first = malloc(sizeof(orc_piece) * cap);
    orc_piece* second = malloc(sizeof(orc_piece) * cap);
    for (int f = 0; f < nflows; ++f) {
        int s = fsrc[f], d = fdst[f], v = fvia[f];
        uint64_t bytes = (uint64_t)fbytes[f];
        uint64_t off = pair_done[s * R + d];
        pair_done[s * R + d] += bytes;
        for (uint64_t o = 0; o < bytes; o += piece) {
            uint64_t n = bytes - o < piece ? bytes - o : piece;
            if (n1 + 1 > cap || n2 + 1 > cap) {
                cap *= 2;
                first = realloc(first, sizeof(orc_piece) * cap);
                second = realloc(second, sizeof(orc_piece) * cap);
            }
            const uint8_t* src = send[s] + sd[s * R + d] + off + o;
            uint8_t* dst = recv[d] + rd[d * R + s] + off + o;
            if (v < 0 || !staging) {
                first[n1++] = (orc_piece){src, dst, n};
            } else {
                uint8_t* st = staging[v] + stage_off[v];
                stage_off[v] += n;
                first[n1++] = (orc_piece){src, st, n};
                second[n2++] = (orc_piece){st, dst, n};
            }
        }
    }
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = malloc(sizeof(pthread_t) * nthreads);
    orc_job* jobs = malloc(sizeof(orc_job) * nthreads);
    double t0 = now_s();
    for (int phase = 0; phase < 2; ++phase) {
        orc_piece* p = phase ? second : first;
        int np = (int)(phase ? n2 : n1);
        if (!np) continue;
        for (int t = 0; t < nthreads; ++t) {
            jobs[t] = (orc_job){p, np, t, nthreads};
            pthread_create(&th[t], NULL, orc_worker, &jobs[t]);
        }
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    }
    double dt = now_s() - t0;
    free(th);
    free(jobs);
    free(first);
    free(second);
    free(sd);
    free(rd);
    free(pair_done);
    free(stage_off);
    return dt;
}
