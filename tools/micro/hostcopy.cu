// Host-side copy rates of the GPU box, for the host-input (e2e) path:
// multi-threaded memcpy into pinned staging (from pageable and from pinned
// sources), cudaMemcpyAsync H2D from pinned and from pageable memory, and a
// pinned DMA running concurrently with host memcpy threads.  One JSON object.
//   nvcc -O3 -std=c++17 -o hostcopy hostcopy.cu -lpthread && ./hostcopy
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

static void par_memcpy(char* dst, const char* src, size_t n, int T) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
        const size_t lo = n * t / T, hi = n * (t + 1) / T;
        th.emplace_back([=] { memcpy(dst + lo, src + lo, hi - lo); });
    }
    for (auto& x : th) x.join();
}

int main() {
    const size_t N = 240ull << 20;
    char* pageable = (char*)malloc(N);
    char* pageable2 = (char*)malloc(N);
    char *pin1, *pin2, *dev;
    cudaMallocHost(&pin1, N);
    cudaMallocHost(&pin2, N);
    cudaMalloc(&dev, N);
    memset(pageable, 1, N);
    memset(pageable2, 1, N);
    memset(pin1, 2, N);
    memset(pin2, 3, N);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto best = [&](auto f) {
        double b = 1e30;
        for (int r = 0; r < 5; ++r) {
            const double t0 = now();
            f();
            const double dt = now() - t0;
            if (dt < b) b = dt;
        }
        return N / b / 1e9;
    };
    printf("{\"bytes\": %zu, \"hw_threads\": %u", N, std::thread::hardware_concurrency());
    for (int T : {1, 2, 4, 8, 12, 16}) {
        printf(", \"memcpy_pageable_to_pinned_T%d\": %.1f", T,
               best([&] { par_memcpy(pin1, pageable, N, T); }));
        printf(", \"memcpy_pinned_to_pinned_T%d\": %.1f", T,
               best([&] { par_memcpy(pin1, pin2, N, T); }));
    }
    printf(", \"h2d_pinned\": %.1f", best([&] {
               cudaMemcpyAsync(dev, pin1, N, cudaMemcpyHostToDevice, s);
               cudaStreamSynchronize(s);
           }));
    printf(", \"h2d_pageable\": %.1f", best([&] {
               cudaMemcpyAsync(dev, pageable, N, cudaMemcpyHostToDevice, s);
               cudaStreamSynchronize(s);
           }));
    // DMA of the first half from pinned while 8 threads memcpy the second half
    for (int T : {4, 8, 16}) {
        printf(", \"dma_half_plus_memcpy_half_T%d\": %.1f", T, best([&] {
                   cudaMemcpyAsync(dev, pin1, N / 2, cudaMemcpyHostToDevice, s);
                   par_memcpy(pin2 + N / 2, pageable2 + N / 2, N / 2, T);
                   cudaStreamSynchronize(s);
               }));
    }
    printf("}\n");
    return 0;
}
