// GPU check: rn_div_inrange (geometry.cuh) equals __ddiv_rn bit for bit on
// random operands inside its domain (|a| >= 2^-900, quotient normal).
// Built by tests/test_gpu_division.py with nvcc (sm_100a).
#include <cstdint>
#include <cuda_runtime.h>
#include "geometry.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}

// operand from a random mantissa, a random exponent in [lo, hi] and a random sign;
// one in eight mantissas is forced near 1 or near 2 (the hardest quotients)
__device__ double operand(uint64_t h, int lo, int hi) {
    uint64_t m = h & 0xfffffffffffffull;
    const int sel = (int)((h >> 52) & 7);
    if (sel == 0) m &= 0xffull;                                   // just above 1
    if (sel == 1) m |= 0xfffffffffff00ull;                        // just below 2
    const int e = lo + (int)(mix(h) % (uint64_t)(hi - lo + 1));
    const uint64_t bits = ((uint64_t)(e + 1023) << 52) | m | ((h >> 63) << 63);
    return __longlong_as_double((long long)bits);
}

__global__ void div_check_kernel(uint64_t n, uint64_t seed, unsigned long long* bad,
                                 unsigned long long* tested, double* first) {
    unsigned long long nb = 0, nt = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h1 = mix(seed ^ (2 * i)), h2 = mix(seed ^ (2 * i + 1));
        const double a = operand(h1, -200, 120);
        const double b = operand(h2, -140, 120);
        const double ref = __ddiv_rn(a, b);
        const double aq = fabs(ref);
        if (!(aq >= 2.2250738585072014e-308) || !(fabs(a) >= 0x1p-900) || isinf(ref)) continue;
        ++nt;
        const double got = bt::rn_div_inrange(a, b);
        if (__double_as_longlong(got) != __double_as_longlong(ref)) {
            if (atomicAdd(bad, 1ull) == 0) {
                first[0] = a;
                first[1] = b;
            }
            ++nb;
        }
    }
    atomicAdd(tested, nt);
}

extern "C" int bt_div_check(unsigned long long n, unsigned long long seed,
                            unsigned long long* out /* bad, tested */, double* first) {
    unsigned long long* d = nullptr;
    double* f = nullptr;
    if (cudaMalloc(&d, 2 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    if (cudaMalloc(&f, 2 * sizeof(double)) != cudaSuccess) return 1;
    cudaMemset(d, 0, 2 * sizeof(unsigned long long));
    cudaMemset(f, 0, 2 * sizeof(double));
    div_check_kernel<<<148 * 8, 256>>>(n, seed, d, d + 1, f);
    if (cudaDeviceSynchronize() != cudaSuccess) return 2;
    cudaMemcpy(out, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemcpy(first, f, 2 * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(f);
    return 0;
}
