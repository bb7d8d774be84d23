/* A caller that used NCCL, switched to include/nimble.h: one process per GPU,
 * a skewed all-to-allv (the reference's gen_skewed_a2av matrix), delivery
 * checked on the device.  Plain C; the only CUDA runtime calls are the device
 * choice and the read-back of the mismatch count.
 *
 *   cc -O2 -I include -I /usr/local/cuda/include examples/alltoallv.c \
 *      -L paper_2604_00317_b200 -lnimble_b200 -L /usr/local/cuda/lib64 -lcudart \
 *      -Wl,-rpath,$PWD/paper_2604_00317_b200 -o alltoallv
 *   RANK=r WORLD_SIZE=n NIMBLE_ID_FILE=/tmp/id ./alltoallv    (one per GPU)
 *
 * The communicator id travels through a file here (MPI_Bcast or a
 * torch.distributed broadcast in a real job), as ncclUniqueId does. */
#include <cuda_runtime.h>
#include <nimble.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define CHECK(call)                                                                 \
    do {                                                                            \
        nimbleResult_t r_ = (call);                                                 \
        if (r_ != nimbleSuccess) {                                                  \
            fprintf(stderr, "%s failed (%d): %s\n", #call, r_, nimbleGetLastError()); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

int main(void) {
    const int rank = env_int("RANK", 0), nranks = env_int("WORLD_SIZE", 1);
    const char* idfile = getenv("NIMBLE_ID_FILE") ? getenv("NIMBLE_ID_FILE") : "/tmp/nimble_example_id";
    cudaSetDevice(env_int("LOCAL_RANK", rank));

    nimbleUniqueId id;
    if (rank == 0) {
        CHECK(nimbleGetUniqueId(&id));
        char tmp[512];
        snprintf(tmp, sizeof tmp, "%s.tmp", idfile);
        FILE* f = fopen(tmp, "wb");
        fwrite(&id, sizeof id, 1, f);
        fclose(f);
        rename(tmp, idfile);
    } else {
        FILE* f = NULL;
        while (!(f = fopen(idfile, "rb"))) usleep(10000);
        if (fread(&id, sizeof id, 1, f) != 1) {
            fprintf(stderr, "rank %d: short id file %s\n", rank, idfile);
            return 1;
        }
        fclose(f);
    }
    nimbleComm_t comm;
    CHECK(nimbleCommInitRank(&comm, nranks, id, rank));

    /* the reference's skewed matrix: 64 MiB per rank, 70% of every rank's data to rank 0 */
    uint64_t* m = calloc((size_t)nranks * nranks, sizeof *m);
    if (nranks > 1) CHECK(nimbleGenSkewed(nranks, 64ull << 20, 0.7, 0, 0, m));
    else m[0] = 64ull << 20; /* one rank: its self segment */
    size_t sc[32], sd[32], rc[32], rd[32], stot = 0, rtot = 0;
    for (int p = 0; p < nranks; ++p) {
        sc[p] = m[(size_t)rank * nranks + p], sd[p] = stot, stot += sc[p];
        rc[p] = m[(size_t)p * nranks + rank], rd[p] = rtot, rtot += rc[p];
    }
    void *send, *recv;
    CHECK(nimbleMemAlloc(&send, stot ? stot : 16));
    CHECK(nimbleMemAlloc(&recv, rtot ? rtot : 16));
    for (int p = 0; p < nranks; ++p) CHECK(nimbleFillPayload((char*)send + sd[p], 0, sc[p], 1, rank, p, NULL));
    void *hs, *hr; /* registration: zero copy, receiver-driven pulls (as ncclCommRegister) */
    CHECK(nimbleCommRegister(comm, send, stot ? stot : 16, &hs));
    CHECK(nimbleCommRegister(comm, recv, rtot ? rtot : 16, &hr));

    for (int it = 0; it < 10; ++it) /* back to back on one stream: the launches chain */
        CHECK(nimbleAlltoAllv(send, sc, sd, recv, rc, rd, nimbleUint8, comm, NULL));

    uint64_t* bad;
    CHECK(nimbleMemAlloc((void**)&bad, sizeof *bad));
    cudaMemset(bad, 0, sizeof *bad);
    for (int p = 0; p < nranks; ++p) CHECK(nimbleCheckPayload((char*)recv + rd[p], 0, rc[p], 1, p, rank, bad, NULL));
    uint64_t host_bad = 0;
    cudaMemcpy(&host_bad, bad, sizeof host_bad, cudaMemcpyDeviceToHost);
    nimbleResult_t async = nimbleSuccess;
    CHECK(nimbleCommGetAsyncError(comm, &async));
    printf("rank %d: received %zu bytes from %d ranks, %llu mismatched, async %d\n", rank, rtot, nranks,
           (unsigned long long)host_bad, (int)async);

    CHECK(nimbleCommDeregister(comm, hs));
    CHECK(nimbleCommDeregister(comm, hr));
    CHECK(nimbleCommDestroy(comm));
    nimbleMemFree(send);
    nimbleMemFree(recv);
    nimbleMemFree(bad);
    free(m);
    if (rank == 0) unlink(idfile);
    return host_bad || async != nimbleSuccess;
}
