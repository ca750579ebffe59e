// multi.cuh -- one handle over several GPUs of one process (SURVEY §8b/§8e,
// PAPER.md:296): particles are sharded in contiguous ranges
// [r*ceil(N/P), (r+1)*ceil(N/P)), the mesh is replicated, every GPU keeps a
// private tally, and once per batch the tallies are summed by one NCCL
// all-reduce over NVLink before the on-device finalize (so every GPU holds
// the batch statistics).  Every call fans out to the shards on one host
// thread per GPU.  NCCL is loaded at run time (dlopen), so the library loads
// without it; device sets with a repeated ordinal (tests on one GPU) or no
// NCCL reduce through peer copies instead.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load() {
        if (lib) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (lib) break;
        }
        if (!lib) return false;
        CommInitAll = (decltype(CommInitAll))dlsym(lib, "ncclCommInitAll");
        CommDestroy = (decltype(CommDestroy))dlsym(lib, "ncclCommDestroy");
        AllReduce = (decltype(AllReduce))dlsym(lib, "ncclAllReduce");
        GroupStart = (decltype(GroupStart))dlsym(lib, "ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))dlsym(lib, "ncclGroupEnd");
        GetErrorString = (decltype(GetErrorString))dlsym(lib, "ncclGetErrorString");
        return CommInitAll && CommDestroy && AllReduce && GroupStart && GroupEnd && GetErrorString;
    }
};
static NcclApi g_nccl;

struct Multi {
    std::vector<bt_tally*> shard;
    std::vector<int64_t> lo, hi;
    std::vector<ncclComm_t> comm;  // empty: peer-copy reduction
    double source_weight = 0.0;    // the batch's recorded weight (global rule)
    int64_t cap = 0;
};

__global__ void add_kernel(double* __restrict__ a, const double* __restrict__ b, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = __dadd_rn(a[i], b[i]);
}

// run fn(r) for every shard on its own host thread; the first failure wins
// and its message is carried to the calling thread
template <class F>
static bt_status fan_out(Multi* m, F fn) {
    const int n = (int)m->shard.size();
    std::vector<bt_status> st((size_t)n, BT_OK);
    std::vector<std::string> msg((size_t)n);
    std::vector<std::thread> th;
    for (int r = 1; r < n; ++r)
        th.emplace_back([&, r] {
            st[(size_t)r] = fn(r);
            if (st[(size_t)r] != BT_OK) msg[(size_t)r] = g_err;
        });
    st[0] = fn(0);
    if (st[0] != BT_OK) msg[0] = g_err;
    for (auto& t : th) t.join();
    for (int r = 0; r < n; ++r)
        if (st[(size_t)r] != BT_OK) {
            g_err = msg[(size_t)r];
            return st[(size_t)r];
        }
    return BT_OK;
}

static void destroy_multi(Multi* m) {
    for (ncclComm_t c : m->comm) g_nccl.CommDestroy(c);
    for (bt_tally* s : m->shard) bt_destroy(s);
    delete m;
}

// sum the shards' batch tallies in place on every GPU
static bt_status multi_reduce(bt_tally* h) {
    Multi* m = h->multi;
    const int n = (int)m->shard.size();
    const size_t nb = (size_t)(h->ne * h->ngroups);
    if (n == 1 && m->comm.empty()) return BT_OK;
    if (!m->comm.empty()) {
        if (g_nccl.GroupStart() != ncclSuccess) return set_err(BT_ECUDA, "ncclGroupStart");
        for (int r = 0; r < n; ++r) {
            bt_tally* s = m->shard[(size_t)r];
            CK(cudaSetDevice(s->dev));
            const ncclResult_t e = g_nccl.AllReduce(s->tally, s->tally, nb, ncclFloat64, ncclSum,
                                                    m->comm[(size_t)r], s->stream);
            if (e != ncclSuccess) {
                g_nccl.GroupEnd();
                return set_err(BT_ECUDA, "ncclAllReduce: %s", g_nccl.GetErrorString(e));
            }
        }
        if (g_nccl.GroupEnd() != ncclSuccess) return set_err(BT_ECUDA, "ncclGroupEnd");
        for (bt_tally* s : m->shard) {
            CK(cudaSetDevice(s->dev));
            CK(cudaStreamSynchronize(s->stream));
        }
    } else {
        // peer copies into shard 0, summed there in shard order, copied back
        bt_tally* s0 = m->shard[0];
        CK(cudaSetDevice(s0->dev));
        double* tmp = nullptr;
        CK(cudaMalloc(&tmp, sizeof(double) * nb));
        for (int r = 1; r < n; ++r) {
            bt_tally* s = m->shard[(size_t)r];
            CK(cudaSetDevice(s->dev));
            CK(cudaStreamSynchronize(s->stream));
            CK(cudaSetDevice(s0->dev));
            CK(cudaMemcpyPeerAsync(tmp, s0->dev, s->tally, s->dev, sizeof(double) * nb, s0->stream));
            add_kernel<<<grid_for((int64_t)nb, 256), 256, 0, s0->stream>>>(s0->tally, tmp,
                                                                          (int64_t)nb);
            CK(cudaGetLastError());
        }
        CK(cudaStreamSynchronize(s0->stream));
        for (int r = 1; r < n; ++r) {
            bt_tally* s = m->shard[(size_t)r];
            CK(cudaMemcpyPeerAsync(s->tally, s->dev, s0->tally, s0->dev, sizeof(double) * nb,
                                   s0->stream));
        }
        CK(cudaStreamSynchronize(s0->stream));
        cudaFree(tmp);
    }
    return BT_OK;
}

// the shard's share [lo, hi) of a call over particles [0, count)
static inline int64_t shard_count(const Multi* m, int r, int64_t count) {
    return std::max<int64_t>(0, std::min(count, m->hi[(size_t)r]) - m->lo[(size_t)r]);
}

static bt_status multi_create(const double* vertices, int64_t num_vertices,
                              const int32_t* elements, const int32_t* adj_elem,
                              const int8_t* adj_face, int64_t num_elements, const double* bbox,
                              const double* centroid0, int64_t num_particles, int32_t num_groups,
                              const int32_t* devices, int32_t ndev, bt_tally** out) {
    Multi* m = new Multi();
    m->cap = num_particles;
    const int64_t per = (num_particles + ndev - 1) / ndev;
    m->shard.assign((size_t)ndev, nullptr);
    for (int r = 0; r < ndev; ++r) {
        m->lo.push_back(std::min<int64_t>(r * per, num_particles));
        m->hi.push_back(std::min<int64_t>((r + 1) * per, num_particles));
    }
    const bt_status s = fan_out(m, [&](int r) {
        const int64_t cap_r = std::max<int64_t>(1, m->hi[(size_t)r] - m->lo[(size_t)r]);
        return bt_create(vertices, num_vertices, elements, adj_elem, adj_face, num_elements, bbox,
                         centroid0, cap_r, num_groups, devices[r], &m->shard[(size_t)r]);
    });
    if (s != BT_OK) {
        const std::string keep = g_err;
        for (bt_tally*& t : m->shard)
            if (t) bt_destroy(t);
        m->shard.clear();
        delete m;
        g_err = keep;
        return s;
    }
    // NCCL over the distinct devices (one communicator per GPU, ncclCommInitAll)
    bool distinct = true;
    for (int i = 0; i < ndev; ++i)
        for (int j = 0; j < i; ++j) distinct &= devices[i] != devices[j];
    // (also for one GPU: the all-reduce is then a copy, but the NCCL path runs)
    if (distinct && g_nccl.load()) {
        m->comm.assign((size_t)ndev, nullptr);
        const ncclResult_t e = g_nccl.CommInitAll(m->comm.data(), ndev, devices);
        if (e != ncclSuccess) {
            m->comm.clear();
            destroy_multi(m);
            return set_err(BT_ECUDA, "ncclCommInitAll: %s", g_nccl.GetErrorString(e));
        }
    } else if (ndev > 1) {
        // peer access where the hardware allows it (NVLink); copies work either way
        for (int i = 0; i < ndev; ++i)
            for (int j = 0; j < ndev; ++j) {
                int ok = 0;
                if (devices[i] != devices[j] &&
                    cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]) == cudaSuccess && ok) {
                    cudaSetDevice(devices[i]);
                    cudaDeviceEnablePeerAccess(devices[j], 0);
                    cudaGetLastError();  // already enabled
                }
            }
    }
    bt_tally* h = new bt_tally();
    bt_tally* s0 = m->shard[0];
    h->dev = s0->dev;
    h->nv = s0->nv;
    h->ne = s0->ne;
    h->cap = num_particles;
    h->ngroups = num_groups;
    h->multi = m;
    *out = h;
    return BT_OK;
}

// ---- the fanned-out calls (h->multi != nullptr)

static bt_status multi_initialize(bt_tally* h, const double* positions, int64_t size,
                                  int32_t mem_kind, int32_t mode, bt_summary* summary) {
    Multi* m = h->multi;
    if (size < 0 || size % 3 != 0)
        return set_err(BT_EINVAL, "positions must hold 3*count floats, got %lld", (long long)size);
    const int64_t count = size / 3;
    if (count > m->cap)
        return set_err(BT_EINVAL, "count %lld exceeds capacity %lld", (long long)count,
                       (long long)m->cap);
    if (mem_kind != BT_MEM_HOST && m->shard.size() > 1)
        return set_err(BT_EINVAL, "a multi-GPU handle takes host arrays");
    std::vector<bt_summary> part(m->shard.size());
    const bt_status s = fan_out(m, [&](int r) {
        const int64_t n = shard_count(m, r, count);
        return bt_initialize_particle_location(m->shard[(size_t)r],
                                               n ? positions + 3 * m->lo[(size_t)r] : positions,
                                               3 * n, mem_kind, mode, &part[(size_t)r]);
    });
    m->source_weight = 0.0;
    if (summary) {
        memset(summary, 0, sizeof *summary);
        for (const bt_summary& p : part) {
            summary->sweeps = std::max(summary->sweeps, p.sweeps);
            summary->events += p.events;
            summary->reached += p.reached;
            summary->boundary_exits += p.boundary_exits;
            summary->stuck_recoveries += p.stuck_recoveries;
            summary->stuck_terminations += p.stuck_terminations;
        }
    }
    return s;
}

static bt_status multi_move(bt_tally* h, const double* destinations, const int8_t* flying,
                            const double* weights, const int32_t* groups, int64_t count,
                            int32_t mem_kind, bt_summary* summary) {
    Multi* m = h->multi;
    if (summary) memset(summary, 0, sizeof *summary);
    if (count < 0 || count > m->cap)
        return set_err(BT_EINVAL, "count %lld outside [0, %lld]", (long long)count,
                       (long long)m->cap);
    if (count == 0) return BT_OK;
    if (mem_kind != BT_MEM_HOST && m->shard.size() > 1)
        return set_err(BT_EINVAL, "a multi-GPU handle takes host arrays");
    if (groups) {  // range check before any shard moves (tally.py:262-266 deviation)
        const int64_t bad = first_bad_group(groups, count, h->ngroups);
        if (bad >= 0)
            return set_err(BT_EINDEX, "group %d out of range [0, %d)", groups[bad], h->ngroups);
    }
    // the batch's source weight: the first move whose flying weight is non-zero,
    // decided on the whole move (tally.py:267-269), summed over the shards
    const bool recording = m->source_weight == 0.0;
    std::vector<bt_summary> part(m->shard.size());
    std::vector<double> w((size_t)m->shard.size(), 0.0);
    const bt_status s = fan_out(m, [&](int r) {
        bt_tally* t = m->shard[(size_t)r];
        const int64_t lo = m->lo[(size_t)r], n = shard_count(m, r, count);
        if (recording) t->source_weight = 0.0;
        if (n == 0) return BT_OK;
        const bt_status st = bt_move_to_next_location(
            t, destinations + 3 * lo, flying + lo, weights + lo, groups ? groups + lo : nullptr,
            n, mem_kind, &part[(size_t)r]);
        w[(size_t)r] = t->source_weight;
        return st;
    });
    if (recording) {
        double tot = 0.0;
        for (double x : w) tot += x;
        m->source_weight = tot;
        if (tot != 0.0)
            for (bt_tally* t : m->shard) t->source_weight = tot;  // stop recording
    }
    if (summary)
        for (const bt_summary& p : part) {
            summary->sweeps = std::max(summary->sweeps, p.sweeps);
            summary->events += p.events;
            summary->reached += p.reached;
            summary->boundary_exits += p.boundary_exits;
            summary->stuck_recoveries += p.stuck_recoveries;
            summary->stuck_terminations += p.stuck_terminations;
        }
    return s;
}

static bt_status multi_finalize(bt_tally* h, double source_weight) {
    Multi* m = h->multi;
    const double w = source_weight > 0.0 ? source_weight : m->source_weight;
    if (!(w > 0.0))
        return set_err(BT_ERUNTIME, "no source weight recorded for this batch; pass source_weight");
    TRY(multi_reduce(h));
    TRY(fan_out(m, [&](int r) { return bt_finalize_batch(m->shard[(size_t)r], w); }));
    m->source_weight = 0.0;
    for (bt_tally* t : m->shard) t->source_weight = 0.0;
    return BT_OK;
}

static bt_status multi_read_tally(bt_tally* h, int32_t which, double* out, int64_t n) {
    Multi* m = h->multi;
    if (n != h->ne * h->ngroups) return set_err(BT_EINVAL, "n must be E*G");
    if (which != BT_TALLY_BATCH || m->shard.size() == 1)
        return bt_read_tally(m->shard[0], which, out, n);  // finalized moments: identical on every GPU
    // the unfinalized batch: per-GPU partials summed on the host in shard order
    std::vector<std::vector<double>> part(m->shard.size());
    TRY(fan_out(m, [&](int r) {
        part[(size_t)r].resize((size_t)n);
        return bt_read_tally(m->shard[(size_t)r], which, part[(size_t)r].data(), n);
    }));
    for (int64_t b = 0; b < n; ++b) {
        double a = part[0][(size_t)b];
        for (size_t r = 1; r < part.size(); ++r) a += part[r][(size_t)b];
        out[b] = a;
    }
    return BT_OK;
}

static bt_status multi_read_particles(bt_tally* h, int64_t count, double* position,
                                      int32_t* element, int8_t* alive, int8_t* entry_face,
                                      int8_t* stuck, int8_t* outcome, double* seg_total) {
    Multi* m = h->multi;
    if (count < 0 || count > m->cap) return set_err(BT_EINVAL, "count out of range");
    return fan_out(m, [&](int r) {
        const int64_t lo = m->lo[(size_t)r], n = shard_count(m, r, count);
        if (n == 0) return BT_OK;
        return bt_read_particles(m->shard[(size_t)r], n, position ? position + 3 * lo : nullptr,
                                 element ? element + lo : nullptr, alive ? alive + lo : nullptr,
                                 entry_face ? entry_face + lo : nullptr,
                                 stuck ? stuck + lo : nullptr, outcome ? outcome + lo : nullptr,
                                 seg_total ? seg_total + lo : nullptr);
    });
}

static bt_status multi_read_digest(bt_tally* h, int64_t count, uint64_t* digest,
                                   int64_t* events) {
    Multi* m = h->multi;
    if (count < 0 || count > m->cap) return set_err(BT_EINVAL, "count out of range");
    return fan_out(m, [&](int r) {
        const int64_t lo = m->lo[(size_t)r], n = shard_count(m, r, count);
        if (n == 0) return BT_OK;
        return bt_read_digest(m->shard[(size_t)r], n, digest ? digest + lo : nullptr,
                              events ? events + lo : nullptr);
    });
}

static bt_status multi_last_timing(bt_tally* h, float* walk_ms, float* call_ms,
                                   int64_t* kernels) {
    Multi* m = h->multi;
    float w = 0.f, c = 0.f;
    int64_t k = 0;
    for (bt_tally* t : m->shard) {
        float w1 = 0.f, c1 = 0.f;
        int64_t k1 = 0;
        TRY(bt_last_timing(t, &w1, &c1, &k1));
        w = std::max(w, w1);
        c = std::max(c, c1);
        k += k1;
    }
    if (walk_ms) *walk_ms = w;
    if (call_ms) *call_ms = c;
    if (kernels) *kernels = k;
    return BT_OK;
}
