// Dependent-latency and throughput probes for the fp64/fp32 ops of the exit filter (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void dfma_lat(double* out, long long* cyc, double a, double b) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void dadd_lat(double* out, long long* cyc, double a, double b) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = __dadd_rn(x, a);
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void ffma_lat(double* out, long long* cyc, double a, double b) {
    float x = (float)out[threadIdx.x]; float fa = (float)a, fb = (float)b;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fmaf(x, fa, fb);
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void f2f_lat(double* out, long long* cyc, double a, double b) {
    double x = out[threadIdx.x];
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) { float f = (float)x; x = (double)f; }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread, many warps
template <int K>
__global__ void dfma_tp(double* out, long long* cyc, double a, double b) {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = out[threadIdx.x] + j;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    long long t1 = clock64();
    double s = 0; for (int j = 0; j < 8; ++j) s += x[j];
    out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void ffma_tp(double* out, long long* cyc, double a, double b) {
    float x[8]; float fa = (float)a, fb = (float)b;
    for (int j = 0; j < 8; ++j) x[j] = (float)out[threadIdx.x] + j;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], fa, fb);
    long long t1 = clock64();
    float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
    out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void f2f_tp(double* out, long long* cyc, double a, double b) {
    double x[8]; float y[8];
    for (int j = 0; j < 8; ++j) { x[j] = out[threadIdx.x] + j; y[j] = 0; }
    long long t0 = clock64();
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) { y[j] += (float)x[j]; x[j] = __dadd_rn(x[j], 1e-300); }
    long long t1 = clock64();
    float s = 0; for (int j = 0; j < 8; ++j) s += y[j];
    out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
typedef void (*K)(double*, long long*, double, double);
int main() {
    double* d; long long* c; cudaMalloc(&d, 1 << 16); cudaMalloc(&c, 8); cudaMemset(d, 0, 1 << 16);
    struct { const char* n; K k; int th; int ops; } ks[] = {
        {"dfma_lat", dfma_lat, 32, 1}, {"dadd_lat", dadd_lat, 32, 1}, {"ffma_lat", ffma_lat, 32, 1},
        {"f2f_roundtrip_lat", f2f_lat, 32, 1},
        {"dfma_tp(1024thr/SM)", dfma_tp<0>, 1024, 8}, {"ffma_tp(1024thr/SM)", ffma_tp, 1024, 8},
        {"f2f+dadd_tp(1024thr/SM)", f2f_tp, 1024, 8}};
    for (auto& k : ks) {
        k.k<<<1, k.th>>>(d, c, 1.0000001, 1e-7); cudaDeviceSynchronize();
        k.k<<<1, k.th>>>(d, c, 1.0000001, 1e-7); cudaDeviceSynchronize();
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        double per = (double)cy / (N * k.ops);
        if (k.th == 32) printf("%-26s %.2f cycles/op (dependent)\n", k.n, per);
        else printf("%-26s %.2f warp-inst/cycle/SM (%d warps)\n", k.n, (k.th / 32.0) / per, k.th / 32);
    }
    return 0;
}
