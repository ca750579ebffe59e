// host_stage.cuh -- host-to-device copies of caller buffers (the host-input
// path of initialize_particle_location / move_to_next_location).
// Part of libb200tally (included by b200tally.cu, one translation unit).
//
// A caller's PINNED buffer is copied by the DMA engine directly.  A PAGEABLE
// buffer (an ordinary numpy array -- what a drop-in user passes) would go
// through the driver's own staging at ~11 GB/s on the GPU box
// (tools/micro/hostcopy.cu, profiles/r02_hostcopy.json); here it is split into
// pieces that a pool of host threads copies into a ring of pinned slots
// (~50 GB/s with 4+ threads) while the DMA engine drains the previous slots
// (53 GB/s): the two overlap, so the transfer runs near PCIe speed.
#pragma once

#include <condition_variable>
#include <functional>
#include <mutex>

// a fixed pool of host threads running one parallel job at a time
class HostPool {
   public:
    explicit HostPool(int n) : n_(std::max(1, n)) {
        for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return n_; }
    // fn(i) for i in [0, size()), the calling thread runs i = 0
    void run(const std::function<void(int)>& fn) {
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            left_ = n_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return left_ == 0; });
        fn_ = nullptr;
    }

   private:
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* f;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                f = fn_;
            }
            (*f)(i);
            {
                std::lock_guard<std::mutex> g(m_);
                if (--left_ == 0) done_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int left_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// true when `p` is ordinary pageable host memory (not registered / pinned)
static bool is_pageable(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// ring of pinned slots + host threads for pageable sources
struct HostStager {
    static constexpr size_t SLOT = 8u << 20;  // bytes per slot
    static constexpr int NSLOT = 8;
    char* ring = nullptr;  // NSLOT * SLOT pinned bytes
    cudaEvent_t ev[NSLOT] = {};
    int next = 0;
    HostPool* pool = nullptr;

    bt_status init() {
        if (ring) return BT_OK;
        CK(cudaMallocHost((void**)&ring, (size_t)NSLOT * SLOT));
        for (cudaEvent_t& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
        // 4 threads reach the host copy bandwidth on the GPU box (hostcopy.cu);
        // copying while the DMA engine also reads host memory needs more
        // (16: 90 GB/s combined, 8: 65, 4: 59)
        pool = new HostPool((int)std::min(16u, hc));
        return BT_OK;
    }
    void release() {
        if (ring) {
            for (int k = 0; k < NSLOT; ++k) cudaEventSynchronize(ev[k]);
            cudaFreeHost(ring);
            for (cudaEvent_t e : ev) cudaEventDestroy(e);
        }
        delete pool;
        ring = nullptr;
        pool = nullptr;
    }
    // enqueue dst <- src (bytes) on `st`; returns once `src` has been read
    bt_status copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
        TRY(init());
        const char* s = static_cast<const char*>(src);
        char* d = static_cast<char*>(dst);
        for (size_t off = 0; off < bytes; off += SLOT) {
            const size_t n = std::min(SLOT, bytes - off);
            const int k = next;
            next = (next + 1) % NSLOT;
            CK(cudaEventSynchronize(ev[k]));  // the slot's previous DMA has drained
            char* slot = ring + (size_t)k * SLOT;
            const int T = n >= (1u << 20) ? pool->size() : 1;
            if (T == 1) {
                memcpy(slot, s + off, n);
            } else {
                pool->run([&](int i) {
                    const size_t lo = n * i / T, hi = n * (i + 1) / T;
                    memcpy(slot + lo, s + off + lo, hi - lo);
                });
            }
            CK(cudaMemcpyAsync(d + off, slot, n, cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(ev[k], st));
        }
        return BT_OK;
    }
};
