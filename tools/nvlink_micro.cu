// NVLink primitive microbenchmark (development aid, 2 GPUs, one process).
// Measures one-way and two-way GB/s of the candidate data-movement primitives
// for the forwarding engine:
//   stg     : local LDG.128 -> remote STG.128 (SIMT push)
//   ldg     : remote LDG.128 -> local STG.128 (SIMT pull)
//   tmapush : local TMA bulk load -> smem -> remote TMA bulk store
//   tmapull : remote TMA bulk load -> smem -> local TMA bulk store
//   ce      : cudaMemcpyPeerAsync (copy engines)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/nvlink_micro tools/nvlink_micro.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            std::exit(1);                                                               \
        }                                                                               \
    } while (0)

__global__ void __launch_bounds__(512) k_simt(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n16) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t step = (size_t)gridDim.x * blockDim.x;
    for (; i + 7 * step < n16; i += 8 * step) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = s[i + u * step];
#pragma unroll
        for (int u = 0; u < 8; ++u) d[i + u * step] = v[u];
    }
    for (; i < n16; i += step) d[i] = s[i];
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Each CTA moves contiguous blocks of `blk` bytes through a ring of NS smem stages.
template <int NS>
__global__ void __launch_bounds__(32) k_tma(const char* s, char* d, size_t bytes, int blk) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[NS];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    const size_t nblk = bytes / blk;
    uint32_t phase[NS] = {};
    int k = 0;
    // blocks handled by this CTA: b = blockIdx.x + j*gridDim.x
    size_t first = blockIdx.x;
    size_t mine = first < nblk ? (nblk - first + gridDim.x - 1) / gridDim.x : 0;
    for (size_t j = 0; j < mine + NS; ++j) {
        if (j >= NS) {  // store block j-NS (its load was issued NS iterations ago)
            const int st = (j - NS) % NS;
            asm volatile(
                "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                    sa(&bar[st])),
                "r"(phase[st]));
            phase[st] ^= 1;
            const size_t b = first + (j - NS) * gridDim.x;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + b * blk),
                         "r"(sa(sm + st * blk)), "r"(blk)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;");
        }
        if (j < mine) {
            const int st = j % NS;
            if (j >= NS) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
            const size_t b = first + j * gridDim.x;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[st])), "r"(blk));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    sa(sm + st * blk)),
                "l"(s + b * blk), "r"(blk), "r"(sa(&bar[st]))
                : "memory");
        }
        (void)k;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

struct Bufs {
    char *src0, *dst0, *src1, *dst1;  // srcX/dstX live on device X
};

static float run(const char* name, int mode, bool two_way, Bufs& b, size_t bytes, int ctas, int blk, int reps,
                 cudaStream_t s0, cudaStream_t s1) {
    auto launch = [&](int dev, cudaStream_t st) {
        // one-way: device 0 -> device 1.  two-way: also device 1 -> device 0.
        const char* lsrc = dev == 0 ? b.src0 : b.src1;
        char* rdst = dev == 0 ? b.dst1 : b.dst0;   // remote destination
        const char* rsrc = dev == 0 ? b.src1 : b.src0;  // remote source (pull)
        char* ldst = dev == 0 ? b.dst0 : b.dst1;
        CK(cudaSetDevice(dev));
        switch (mode) {
        case 0: k_simt<<<ctas, 512, 0, st>>>((const uint4*)lsrc, (uint4*)rdst, bytes / 16); break;
        case 1: k_simt<<<ctas, 512, 0, st>>>((const uint4*)rsrc, (uint4*)ldst, bytes / 16); break;
        case 2: k_tma<4><<<ctas, 32, 4 * blk, st>>>(lsrc, rdst, bytes, blk); break;
        case 3: k_tma<4><<<ctas, 32, 4 * blk, st>>>(rsrc, ldst, bytes, blk); break;
        case 4: CK(cudaMemcpyPeerAsync(rdst, dev ^ 1, lsrc, dev, bytes, st)); break;
        }
    };
    cudaEvent_t e0, e1;
    CK(cudaSetDevice(0));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 2; ++w) {
        launch(0, s0);
        if (two_way) launch(1, s1);
    }
    CK(cudaSetDevice(0));
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(1));
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(e0, s0));
    for (int r = 0; r < reps; ++r) {
        launch(0, s0);
        if (two_way) launch(1, s1);
    }
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(e1, s0));
    CK(cudaEventSynchronize(e1));
    CK(cudaSetDevice(1));
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(0));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const float gbps = bytes * (double)reps / (ms * 1e-3) / 1e9;
    std::printf("%-8s %s ctas=%4d blk=%6d : %7.1f GB/s per direction\n", name, two_way ? "2way" : "1way", ctas, blk,
                gbps);
    return gbps;
}

// Incast: GPUs 1..n-1 -> GPU 0, 3*256 MiB total; push (senders STG/TMA store),
// pull (GPU 0 TMA-loads from each peer), ce (senders' copy engines).
static void incast(int n) {
    const size_t per = 256ull << 20;
    std::vector<char*> src(n), dst(n);
    std::vector<cudaStream_t> st(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        for (int p = 0; p < n; ++p)
            if (p != d) {
                cudaError_t e = cudaDeviceEnablePeerAccess(p, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            }
        CK(cudaMalloc(&src[d], per));
        CK(cudaMalloc(&dst[d], per * n));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
        CK(cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 49152));
    }
    for (int mode = 0; mode < 6; ++mode) {
        for (int ctas : {37, 74, 148}) {
            auto go = [&]() {
                for (int s = 1; s < n; ++s) {
                    if (mode == 0) {
                        CK(cudaSetDevice(s));
                        k_simt<<<ctas, 512, 0, st[s]>>>((const uint4*)src[s], (uint4*)(dst[0] + s * per), per / 16);
                    } else if (mode == 1) {
                        CK(cudaSetDevice(s));
                        k_tma<4><<<ctas, 32, 4 * 32768, st[s]>>>(src[s], dst[0] + s * per, per, 32768);
                    } else if (mode == 2) {
                        CK(cudaSetDevice(0));
                        k_tma<4><<<ctas / (n - 1) + 1, 32, 4 * 32768, st[0]>>>(src[s], dst[0] + s * per, per, 32768);
                    } else if (mode == 3) {
                        CK(cudaSetDevice(s));
                        CK(cudaMemcpyPeerAsync(dst[0] + s * per, 0, src[s], s, per, st[s]));
                    } else {  // mixed: sender pushes a share, GPU 0 pulls the rest, concurrently
                        const size_t push = mode == 4 ? per / 2 : per / 4;
                        CK(cudaSetDevice(s));
                        k_tma<4><<<ctas, 32, 4 * 32768, st[s]>>>(src[s], dst[0] + s * per, push, 32768);
                        CK(cudaSetDevice(0));
                        k_tma<4><<<ctas / (n - 1) + 1, 32, 4 * 32768, st[0]>>>(src[s] + push, dst[0] + s * per + push,
                                                                               per - push, 32768);
                    }
                }
            };
            go();
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaDeviceSynchronize());
            }
            auto t0 = std::chrono::steady_clock::now();
            const int reps = 10;
            for (int r = 0; r < reps; ++r) go();
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaDeviceSynchronize());
            }
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            const char* nm[] = {"push-stg", "push-tma", "pull-tma", "ce", "mix50", "mix25"};
            std::printf("incast %d->1 %-9s ctas=%3d : %7.1f GB/s into GPU0\n", n - 1, nm[mode], ctas,
                        per * (double)(n - 1) * reps / s / 1e9);
            if (mode == 3) break;
        }
    }
}

int main(int argc, char** argv) {
    const size_t bytes = 256ull << 20;
    if (argc > 1 && argv[1][0] == 'o') {  // once per primitive, one way 0 -> 1 (for ncu)
        Bufs b{};
        for (int dev = 0; dev < 2; ++dev) {
            CK(cudaSetDevice(dev));
            CK(cudaDeviceEnablePeerAccess(dev ^ 1, 0));
            CK(cudaMalloc(dev ? &b.src1 : &b.src0, bytes));
            CK(cudaMalloc(dev ? &b.dst1 : &b.dst0, bytes));
            CK(cudaMemset(dev ? b.src1 : b.src0, 1, bytes));
            CK(cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 49152));
        }
        CK(cudaSetDevice(0));
        k_simt<<<148, 512>>>((const uint4*)b.src0, (uint4*)b.dst1, bytes / 16);              // push STG
        k_tma<4><<<148, 32, 4 * 32768>>>(b.src0, b.dst1, bytes, 32768);                      // push TMA
        k_tma<4><<<148, 32, 4 * 32768>>>(b.src1, b.dst0, bytes, 32768);                      // pull TMA
        k_simt<<<148, 512>>>((const uint4*)b.src1, (uint4*)b.dst0, bytes / 16);              // pull LDG
        CK(cudaDeviceSynchronize());
        std::printf("once done\n");
        return 0;
    }
    if (argc > 1 && argv[1][0] == 'i') {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        incast(n);
        return 0;
    }
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) {
        std::printf("need 2 GPUs\n");
        return 1;
    }
    Bufs b{};
    cudaStream_t s0, s1;
    for (int dev = 0; dev < 2; ++dev) {
        CK(cudaSetDevice(dev));
        CK(cudaDeviceEnablePeerAccess(dev ^ 1, 0));
        CK(cudaMalloc(dev ? &b.src1 : &b.src0, bytes));
        CK(cudaMalloc(dev ? &b.dst1 : &b.dst0, bytes));
        CK(cudaMemset(dev ? b.src1 : b.src0, 1, bytes));
        CK(cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 49152));
    }
    CK(cudaSetDevice(0));
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaSetDevice(1));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    const int reps = 10;
    for (int tw = 0; tw < 2; ++tw) {
        run("ce", 4, tw, b, bytes, 0, 0, reps, s0, s1);
        for (int ctas : {32, 74, 148, 296}) run("stg", 0, tw, b, bytes, ctas, 0, reps, s0, s1);
        for (int ctas : {32, 74, 148, 296}) run("ldg", 1, tw, b, bytes, ctas, 0, reps, s0, s1);
        for (int blk : {16384, 32768, 49152})
            for (int ctas : {32, 74, 148, 296}) run("tmapush", 2, tw, b, bytes, ctas, blk, reps, s0, s1);
        for (int blk : {16384, 32768, 49152})
            for (int ctas : {32, 74, 148, 296}) run("tmapull", 3, tw, b, bytes, ctas, blk, reps, s0, s1);
    }
    return 0;
}
