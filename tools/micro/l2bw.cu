// L2 bandwidth of this B200 (the roofline denominator for the L2-resident
// walk): streaming 16-byte loads and random 32-byte-sector gathers over a
// buffer that fits in L2 (ld.global.cg: cached in L2 only, so every load is
// an L2 transaction), plus the HBM stream over a buffer far larger than L2
// for comparison.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu && ./l2bw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                \
            return 1;                                                              \
        }                                                                          \
    } while (0)

__device__ __forceinline__ int4 ld_cg(const int4* p) {
    int4 v;
    asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// every thread streams 16-byte words, grid-stride, `reps` passes
__global__ void stream_kernel(const int4* __restrict__ buf, size_t n16, int reps, int* sink) {
    int acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
            const int4 v = ld_cg(buf + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x7fffffff) *sink = acc;
}

// random 32-byte sectors (two 16-byte loads each), 8 independent chains/thread
__global__ void gather_kernel(const int4* __restrict__ buf, uint32_t nsec, int iters, int* sink) {
    uint32_t s[8];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = (t * 8 + k) * 2654435761u + 12345u;
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            s[k] = s[k] * 1664525u + 1013904223u;
            const int4* p = buf + 2 * (size_t)(s[k] % nsec);
            const int4 a = ld_cg(p);
            const int4 b = ld_cg(p + 1);
            acc ^= a.x ^ b.w;
        }
    }
    if (acc == 0x7fffffff) *sink = acc;
}

// random 32-byte sectors, one 256-bit load each (LDG.E.256)
__global__ void gather256_kernel(const int4* __restrict__ buf, uint32_t nsec, int iters, int* sink) {
    uint32_t s[8];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = (t * 8 + k) * 2654435761u + 12345u;
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            s[k] = s[k] * 1664525u + 1013904223u;
            const int4* p = buf + 2 * (size_t)(s[k] % nsec);
            int a0, a1, a2, a3, a4, a5, a6, a7;
            asm volatile("ld.global.cg.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3), "=r"(a4), "=r"(a5), "=r"(a6),
                           "=r"(a7)
                         : "l"(p));
            acc ^= a0 ^ a7;
        }
    }
    if (acc == 0x7fffffff) *sink = acc;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const size_t small = 48ull << 20, big = 4ull << 30;
    int4* buf = nullptr;
    int* sink = nullptr;
    CK(cudaMalloc(&buf, big));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(buf, 1, big));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto best = [&](auto launch, double bytes) -> double {
        float bestms = 1e30f;
        for (int rep = 0; rep < 7; ++rep) {
            launch();
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < bestms) bestms = ms;
        }
        return bytes / (bestms * 1e-3) / 1e9;
    };
    const int threads = 512;
    const int blocks = sms * 4;
    const int reps = 40;
    const double l2_stream = best([&] { stream_kernel<<<blocks, threads>>>(buf, small / 16, reps, sink); },
                                  (double)small * reps);
    const double hbm_stream = best([&] { stream_kernel<<<blocks, threads>>>(buf, big / 16, 1, sink); },
                                   (double)big);
    const int iters = 64;
    const uint32_t nsec = (uint32_t)(small / 32);
    const double l2_gather = best([&] { gather_kernel<<<blocks, threads>>>(buf, nsec, iters, sink); },
                                  (double)blocks * threads * iters * 8 * 32);
    const double l2_gather256 = best([&] { gather256_kernel<<<blocks, threads>>>(buf, nsec, iters, sink); },
                                     (double)blocks * threads * iters * 8 * 32);
    const uint32_t nsec_big = (uint32_t)(big / 32);
    const double hbm_gather = best([&] { gather_kernel<<<blocks, threads>>>(buf, nsec_big, iters, sink); },
                                   (double)blocks * threads * iters * 8 * 32);
    CK(cudaGetLastError());
    int clk = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    printf("{\"sms\": %d, \"l2_bytes\": %d, \"sm_clock_khz_max\": %d, "
           "\"l2_stream_gbs\": %.1f, \"l2_gather32_gbs\": %.1f, \"l2_gather32_v8_gbs\": %.1f, "
           "\"hbm_stream_gbs\": %.1f, \"hbm_gather32_gbs\": %.1f, "
           "\"buffer_l2_mb\": %zu, \"buffer_hbm_mb\": %zu, "
           "\"method\": \"ld.global.cg (L2 only), best of 7, CUDA events; stream = 16 B/thread "
           "grid-stride, gather = random 32 B sectors, 8 chains/thread\"}\n",
           sms, l2, clk, l2_stream, l2_gather, l2_gather256, hbm_stream, hbm_gather, small >> 20, big >> 20);
    return 0;
}
