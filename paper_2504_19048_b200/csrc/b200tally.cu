// b200tally.cu -- B200-native (sm_100a) tet-mesh walk with track-length
// tallies behind the C ABI declared in include/b200tally.h: the handle, the
// host-side move / localization pipelines and every exported entry point.
// The device code lives in the csrc/*.cuh headers of this translation unit.
//
// Replaces the reference's numba hot path:
//   _sweep_fused + trace_and_score  search.py:169-275, 492-517 -> walk_staged_kernel (walk.cuh)
//   _compact_flying + load_step     search.py:160-166,
//                                   particles.py:57-89          -> stage_kernel (walk.cuh)
//   initialize_locations            search.py:557-601          -> locate_grid_kernel (locate.cuh)
//                                                                 (or walk + tiebreak_kernel)
//   _tie_break_faces                search.py:520-551          -> tiebreak_kernel
//   _finalize                       tally.py:83-95              -> finalize_kernel (move_prep.cuh)
//
// Design: persistent CTAs, one particle per lane run to
// completion; warps refill idle lanes from per-warp stages claimed straight
// from the particle arrays (or from the stage kernel's compacted work list),
// so lanes stay busy despite the exponential crossings-per-move tail; the
// exit search is decided by an fp32 filter with proven margins (fp64
// reference arithmetic otherwise); each lane keeps its element's four fp64
// vertices in shared-memory slots, and a crossing fetches only the
// neighbour's one new vertex, named (with the neighbour's vertex order) by a
// 32-byte crossing record per element; tallies are fp64 atomics into a
// private per-GPU grid, warp-aggregated with __match_any_sync where lanes
// score the same bins.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "../../include/b200tally.h"
#include "geometry.cuh"

using namespace bt;

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;

static bt_status set_err(bt_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            bt_status s_ = (e_ == cudaErrorMemoryAllocation) ? BT_ENOMEM : BT_ECUDA;      \
            return set_err(s_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                           __FILE__, __LINE__);                                           \
        }                                                                                 \
    } while (0)


#include "layout.cuh"
#include "walk.cuh"
#include "glibc_math.cuh"
#include "transport.cuh"
#include "sweep.cuh"
#include "locate.cuh"
#include "move_prep.cuh"
#include "adjacency.cuh"

// ---------------------------------------------------------------------------
// handle

struct HostStager;
struct Multi;

struct bt_tally {
    int dev = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;   // kernels
    cudaStream_t cstream = nullptr;  // host-to-device copies (overlap with kernels)
    cudaStream_t stream2 = nullptr;  // odd chunks of a pipelined move (overlap the tails)
    cudaEvent_t ev_s1 = nullptr, ev_s2 = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
    cudaEvent_t evc0 = nullptr, evc1 = nullptr, ev_loc = nullptr;
    cudaEvent_t evchunk[MAX_CHUNKS] = {};
    double* init_stage = nullptr;    // (N,3) localization targets (host inputs)
    int64_t nv = 0, ne = 0, cap = 0;
    int32_t ngroups = 1;
    double bbox[6];
    double c0[3];
    // mesh
    ElemRec* rec = nullptr;
    Vtx* vtx = nullptr;
    XRec* xrec = nullptr;  // crossing records (walk)
    unsigned* xsel = nullptr;  // meshes of >= 2^24 vertices only
    // grid
    GridDev grid{};
    int* cell_start = nullptr;
    int* cand = nullptr;
    ElemLam* lam = nullptr;
    int64_t grid_m = 0;
    // particles (persistent)
    double* pos = nullptr;
    int32_t* element = nullptr;
    int8_t* alive = nullptr;
    int8_t* entry = nullptr;
    int8_t* stuck = nullptr;
    int8_t* outcome = nullptr;
    double* seg_total = nullptr;
    int32_t* group = nullptr;
    // per-move staging
    double* dest = nullptr;
    int8_t* fly = nullptr;
    double* weight = nullptr;
    uint64_t* digest = nullptr;
    int64_t* dcount = nullptr;
    // ordering
    int32_t* order = nullptr;
    unsigned* sort_keys_in = nullptr;
    unsigned* sort_keys_out = nullptr;
    int32_t* sort_vals_in = nullptr;
    void* sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    // tallies
    double* tally = nullptr;
    double* sum = nullptr;
    double* sum_sq = nullptr;
    int64_t batches = 0;
    double source_weight = 0.0;
    // counters
    unsigned long long* dcounters = nullptr;  // queue + counters + flags
    double* wsel = nullptr;                   // device source weight: selected weights
    double* wsel_vals = nullptr;              // pairwise tree nodes
    unsigned* wsel_ticks = nullptr;
    void* wsel_tmp = nullptr;
    size_t wsel_tmp_bytes = 0;
    int wsel_depth = 0;
    unsigned long long* hcounters = nullptr;  // pinned
    int move_chunks = 0;                      // host-input pipeline depth (0 = auto)
    int locate_lanes = 0;                     // grid search lanes per particle (0 = default)
    std::vector<double> host_sel;             // host scratch: weights of flying particles
    HostStager* stager = nullptr;             // pageable host inputs (host_stage.cuh)
    Multi* multi = nullptr;                   // non-null: a multi-GPU handle (multi.cuh)
    bt_mesh* host_mesh = nullptr;             // owned host copy (bt_create_from_mesh / _file)
    // Deferred localization of host positions (initialize -> the next move):
    // positions split into chunks of di_chunk particles; a chunk is either
    // copied and localized already (di_state 0: the DMA read it straight from
    // the caller's pinned buffer during the initialize call) or parked in the
    // pinned host buffer pos_stage (di_state 1) by host threads, to be copied
    // and localized when the move reaches it.
    cudaStream_t lstream = nullptr;           // localization of deferred chunks
    double* pos_stage = nullptr;              // pinned, 3 * cap doubles (lazily)
    int64_t di_count = 0, di_chunk = 0;
    int di_nch = 0;
    bool di_pending = false;
    std::vector<uint8_t> di_state;
    std::vector<cudaEvent_t> di_ev;           // per chunk: localized (on lstream)
    std::vector<cudaEvent_t> di_cev;          // per chunk: copied (on cstream)
    // transport (allocated on first bt_transport_run)
    double* col_tally = nullptr;
    double* col_sum = nullptr;
    double* col_sum_sq = nullptr;
    double* tr_dir = nullptr;
    double* tr_weight = nullptr;
    uint32_t* tr_rng = nullptr;
    unsigned* tr_round_max = nullptr;
    unsigned long long* tr_count = nullptr;  // [0] collisions [1] sweeps [2] alive
    double* tr_wsum = nullptr;               // [0] leaked [1] absorbed [2] stuck [3] track
    double* tr_xs = nullptr;                 // sigma_t | scatter_prob | group_cdf
    int64_t col_batches = 0;
    // Listing-1 callback path
    SweepBufs sb{};
    void* sb_mem = nullptr;
    int8_t* tr_fly = nullptr;     // persistent flying flags of the loaded step
    int32_t* sb_flag = nullptr;   // (cap + 1)
    void* sb_tmp = nullptr;
    size_t sb_tmp_bytes = 0;
    int64_t loaded = 0;           // count of the last bt_load_step
    int64_t tr_sweeps = 0, tr_events = 0, tr_limit = 0, tr_nev = 0;
    bool tr_score = true;
    // snapshot
    double* snap_pos = nullptr;
    int32_t* snap_element = nullptr;
    int8_t* snap_flags = nullptr;  // alive, entry, stuck, outcome (4 x cap)
    double* snap_seg = nullptr;
    bool have_snapshot = false;
    // options
    int64_t max_sweeps = -1;
    bool opt_digest = false;
    bool opt_sort = false;
    int opt_wagg = WAGG_ADAPTIVE;
    bool opt_exact_only = false;
    struct Occ {
        const void* k;
        size_t dyn;
        int bps;
    };
    std::vector<Occ> occ;  // launch_walk's occupancy per (kernel, dynamic shared size)
    bool opt_no_defer = true;  // BT_OPT_DEFER_INIT = 0 (default: measured slower, see below)
    int opt_staged = 2;  // 0: v1 refill, 1: stage kernel + work list, 2: direct refill
    bool opt_stream_move = true;        // BT_OPT_STREAM_MOVE
    unsigned long long* ready = nullptr;  // streamed move: particles landed so far
    int stream_ops = -1;                // stream memory writes usable: -1 unknown, 0 no, 1 yes
    WorkSoA work{};
    void* work_mem = nullptr;
    int blocks_per_sm = 0;
    // timing
    float walk_ms = 0.f, call_ms = 0.f;
    bool call_pending = false;  // ev2..ev3 of an asynchronous call not yet read
    bool walk_first = false;    // ev0 not yet recorded for this move
    int64_t kernels = 0;
};

static bt_status ensure_device(bt_tally* h) {
    CK(cudaSetDevice(h->dev));
    return BT_OK;
}

#define TRY(x)                         \
    do {                               \
        bt_status s__ = (x);           \
        if (s__ != BT_OK) return s__;  \
    } while (0)

#include "host_stage.cuh"

// cuStreamWriteValue64 through the runtime's driver entry point (no link
// against libcuda): the copy engine's front end writes the value once the
// stream's earlier copies are complete, with no SM involved -- the walk that
// waits for it holds every SM.
typedef int (*WriteValue64Fn)(cudaStream_t, unsigned long long, unsigned long long, unsigned);
static WriteValue64Fn write_value64() {
    static WriteValue64Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<WriteValue64Fn>(p);
    }();
    return fn;
}
static bool stream_write(bt_tally* h, unsigned long long* where, unsigned long long v,
                         cudaStream_t st) {
    WriteValue64Fn fn = write_value64();
    return fn && fn(st, (unsigned long long)(uintptr_t)where, v, 0) == 0;
}

// host -> device copy of a caller buffer on `st`: DMA straight from pinned
// memory, through the pinned ring + host threads from pageable memory.
// Returns once `src` has been read.
static bt_status h2d(bt_tally* h, void* dst, const void* src, size_t bytes, cudaStream_t st,
                     bool pageable) {
    if (!bytes) return BT_OK;
    if (!pageable) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return BT_OK;
    }
    if (!h->stager) h->stager = new HostStager();
    return h->stager->copy(dst, src, bytes, st);
}

static bt_status free_all(bt_tally* h) {
    void* ptrs[] = {h->rec, h->vtx, h->xrec, h->xsel, h->cell_start, h->cand, h->lam, h->pos, h->element, h->alive,
                    h->entry, h->stuck, h->outcome, h->seg_total, h->group, h->dest, h->fly,
                    h->weight, h->digest, h->dcount, h->order, h->sort_keys_in,
                    h->sort_keys_out, h->sort_vals_in, h->sort_tmp, h->tally, h->sum,
                    h->sum_sq, h->dcounters, h->wsel, h->wsel_vals, h->wsel_ticks, h->wsel_tmp, h->snap_pos, h->snap_element,
                    h->snap_flags, h->snap_seg, h->work_mem, h->init_stage,
                    h->col_tally, h->col_sum, h->col_sum_sq, h->tr_dir, h->tr_weight,
                    h->tr_rng, h->tr_round_max, h->tr_count, h->tr_wsum, h->tr_xs,
                    h->sb_mem, h->tr_fly, h->sb_flag, h->sb_tmp, h->ready};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->hcounters) cudaFreeHost(h->hcounters);
    if (h->host_mesh) {
        delete h->host_mesh;
        h->host_mesh = nullptr;
    }
    if (h->stager) {
        h->stager->release();
        delete h->stager;
        h->stager = nullptr;
    }
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->ev2) cudaEventDestroy(h->ev2);
    if (h->ev3) cudaEventDestroy(h->ev3);
    if (h->evc0) cudaEventDestroy(h->evc0);
    if (h->evc1) cudaEventDestroy(h->evc1);
    if (h->ev_loc) cudaEventDestroy(h->ev_loc);
    for (cudaEvent_t e : h->evchunk)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : h->di_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : h->di_cev) cudaEventDestroy(e);
    if (h->lstream) cudaStreamDestroy(h->lstream);
    if (h->pos_stage) cudaFreeHost(h->pos_stage);
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->cstream) cudaStreamDestroy(h->cstream);
    if (h->stream2) cudaStreamDestroy(h->stream2);
    if (h->ev_s1) cudaEventDestroy(h->ev_s1);
    if (h->ev_s2) cudaEventDestroy(h->ev_s2);
    return BT_OK;
}

template <typename T>
static bt_status dalloc(T** p, int64_t n) {
    CK(cudaMalloc((void**)p, sizeof(T) * (size_t)std::max<int64_t>(n, 1)));
    return BT_OK;
}

static inline unsigned grid_for(int64_t n, int threads) {
    return (unsigned)std::max<int64_t>(1, (n + threads - 1) / threads);
}

static bt_status build_grid(bt_tally* h) {
    // cells ~ density x E over the bounding box, per-axis counts proportional to extent
    double ext[3];
    double vol = 1.0;
    for (int k = 0; k < 3; ++k) {
        ext[k] = h->bbox[3 + k] - h->bbox[k];
        if (!(ext[k] > 0.0)) ext[k] = 1e-300;
    }
    double maxext = std::max(ext[0], std::max(ext[1], ext[2]));
    for (int k = 0; k < 3; ++k) vol *= std::max(ext[k], 1e-6 * maxext);
    // cells per element (experiments: B200TALLY_GRID_DENSITY).  With the
    // pruned lists, 4 cells per element: 1.24 ms per 1e7 points on C2, 1.58 ms
    // on the 10.1M-tet cube (0.5: 1.85 / 2.50 ms; box lists at 0.5, round 1:
    // 2.85 / 3.62 ms), ~27 list entries per element (profiles/r02_locate.jsonl)
    double density = 4.0;
    if (const char* env = getenv("B200TALLY_GRID_DENSITY")) density = std::max(1e-3, atof(env));
    double target = std::max(1.0, (double)h->ne * density);
    target = std::min(target, (double)(1 << 26));
    double cell = std::cbrt(vol / target);
    GridDev G{};
    // element-cell lists pruned by the barycentric half-spaces (locate.cuh);
    // B200TALLY_GRID_PRUNE=0 lists every bounding-box cell (tests, experiments)
    const char* pe = getenv("B200TALLY_GRID_PRUNE");
    G.prune = pe ? atoi(pe) != 0 : 1;
    int64_t ncells = 1;
    for (int k = 0; k < 3; ++k) {
        int d = (int)std::max(1.0, std::min(4096.0, std::round(ext[k] / cell)));
        if (ext[k] <= 1e-300) d = 1;
        G.dims[k] = d;
        G.org[k] = h->bbox[k];
        G.cs[k] = (ext[k] > 1e-300) ? ext[k] / d : 1.0;
        ncells *= d;
    }
    long long* counts = nullptr;  // 64-bit: the scan accumulates in the input type
    long long* offs = nullptr;
    TRY(dalloc(&counts, h->ne + 1));
    TRY(dalloc(&offs, h->ne + 1));
    CK(cudaMemsetAsync(counts + h->ne, 0, sizeof(long long), h->stream));
    TRY(dalloc(&h->lam, h->ne));
    elem_cells_count_kernel<<<grid_for(h->ne, 256), 256, 0, h->stream>>>(h->rec, h->vtx, h->ne,
                                                                         G, counts);
    CK(cudaGetLastError());
    elem_lambda_kernel<<<grid_for(h->ne, 256), 256, 0, h->stream>>>(h->rec, h->vtx, h->ne, h->lam);
    CK(cudaGetLastError());
    size_t tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offs, (int)(h->ne + 1),
                                     h->stream));
    void* tmp = nullptr;
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offs, (int)(h->ne + 1), h->stream));
    long long m64 = 0;
    CK(cudaMemcpyAsync(&m64, offs + h->ne, sizeof m64, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(tmp);
    if (m64 >= (1ll << 31)) {
        cudaFree(counts);
        cudaFree(offs);
        return set_err(BT_ENOMEM, "localization grid: %lld cell entries exceed 2^31 (lower "
                       "B200TALLY_GRID_DENSITY)", m64);
    }
    const int m = (int)m64;
    unsigned long long *keys = nullptr, *keys_out = nullptr;
    TRY(dalloc(&keys, m));
    TRY(dalloc(&keys_out, m));
    elem_cells_emit_kernel<<<grid_for(h->ne, 256), 256, 0, h->stream>>>(h->ne, G, h->rec, h->vtx,
                                                                        offs, keys);
    CK(cudaGetLastError());
    int cell_bits = 1;
    while ((1ll << cell_bits) < ncells + 1) ++cell_bits;
    tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys_out, m, 0, 32 + cell_bits,
                                      h->stream));
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, keys_out, m, 0, 32 + cell_bits,
                                      h->stream));
    TRY(dalloc(&h->cell_start, ncells + 1));
    TRY(dalloc(&h->cand, m));
    int64_t nthreads = std::max<int64_t>(m, ncells + 1);
    cell_start_kernel<<<grid_for(nthreads, 256), 256, 0, h->stream>>>(keys_out, m, ncells,
                                                                      h->cell_start, h->cand);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(tmp);
    cudaFree(keys);
    cudaFree(keys_out);
    cudaFree(counts);
    cudaFree(offs);
    G.cell_start = h->cell_start;
    G.cand = h->cand;
    h->grid = G;
    h->grid_m = m;
    return BT_OK;
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum_DOUBLE), so the recorded source weight equals the reference's
// `weight[:count][flying].sum()` (tally.py:267-269) bit for bit.
static double pairwise_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

// The same summation tree with its top `depth` levels' left subtrees on
// their own threads: bit-identical to pairwise_sum.
static double pairwise_sum_par(const double* a, int64_t n, int depth) {
    if (depth <= 0 || n <= (1 << 16)) return pairwise_sum(a, n);
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    double left = 0.0;
    std::thread t([&] { left = pairwise_sum_par(a, n2, depth - 1); });
    const double right = pairwise_sum_par(a + n2, n - n2, depth - 1);
    t.join();
    return left + right;
}

// index of the first group id outside [0, ngroups), or -1; blocks on threads
static int64_t first_bad_group(const int32_t* g, int64_t n, int32_t ngroups) {
    const int nt = (int)std::max<int64_t>(
        1, std::min<int64_t>(std::min(8u, std::max(1u, std::thread::hardware_concurrency())),
                             n >> 16));
    std::vector<int64_t> first((size_t)nt, -1);
    auto scan = [&](int b) {
        const int64_t lo = n * b / nt, hi = n * (b + 1) / nt;
        for (int64_t i = lo; i < hi; ++i)
            if ((uint32_t)g[i] >= (uint32_t)ngroups) {
                first[(size_t)b] = i;
                return;
            }
    };
    std::vector<std::thread> th;
    for (int b = 1; b < nt; ++b) th.emplace_back(scan, b);
    scan(0);
    for (auto& t : th) t.join();
    for (int64_t f : first)
        if (f >= 0) return f;
    return -1;
}

// weights[flying != 0] (numpy boolean-mask order) into `out`, in parallel
// blocks; returns the selected count, or -1 (out untouched) when every
// particle is flying and the weights can be summed in place
static int64_t select_flying(const double* w, const int8_t* fly, int64_t n, double* out,
                             int nthreads) {
    const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(nthreads, n >> 16));
    std::vector<int64_t> cnt((size_t)nb + 1, 0);
    auto count_block = [&](int64_t b) {
        const int64_t lo = n * b / nb, hi = n * (b + 1) / nb;
        int64_t c = 0;
        for (int64_t i = lo; i < hi; ++i) c += fly[i] != 0;
        cnt[(size_t)b + 1] = c;
    };
    {
        std::vector<std::thread> th;
        for (int64_t b = 1; b < nb; ++b) th.emplace_back(count_block, b);
        count_block(0);
        for (auto& t : th) t.join();
    }
    for (int64_t b = 0; b < nb; ++b) cnt[(size_t)b + 1] += cnt[(size_t)b];
    if (cnt[(size_t)nb] == n) return -1;
    auto copy_block = [&](int64_t b) {
        const int64_t lo = n * b / nb, hi = n * (b + 1) / nb;
        double* o = out + cnt[(size_t)b];
        for (int64_t i = lo; i < hi; ++i)
            if (fly[i] != 0) *o++ = w[i];
    };
    std::vector<std::thread> th;
    for (int64_t b = 1; b < nb; ++b) th.emplace_back(copy_block, b);
    copy_block(0);
    for (auto& t : th) t.join();
    return cnt[(size_t)nb];
}


#include "multi.cuh"
#include "mesh_io.cuh"

// score_track_length / score_collision (tally.py:67-80) over n events:
// tally[e*G + g] += w * x (kind 0) or w / x (kind 1); flags bit 1: a bin out
// of range, bit 2: sigma_t <= 0 (checked before any score lands)
__global__ void score_check_kernel(const int32_t* __restrict__ el, const int32_t* __restrict__ gr,
                                   const double* __restrict__ x, int64_t n, int64_t ne,
                                   int32_t ng, int kind, unsigned long long* flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (el[i] < 0 || el[i] >= ne || gr[i] < 0 || gr[i] >= ng) atomicOr(flags, 1ull);
    if (kind == 1 && !(x[i] > 0.0)) atomicOr(flags, 2ull);
}
__global__ void score_kernel(const int32_t* __restrict__ el, const int32_t* __restrict__ gr,
                             const double* __restrict__ w, const double* __restrict__ x,
                             int64_t n, int32_t ng, int kind, double* __restrict__ tally) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = kind == 0 ? __dmul_rn(w[i], x[i]) : __ddiv_rn(w[i], x[i]);
    atomicAdd(tally + (int64_t)el[i] * ng + gr[i], v);
}

// single-GPU-only entry points on a multi-GPU handle: forwarded to its one
// shard, refused with several
#define MULTI_SINGLE(h)                                                                    \
    do {                                                                                   \
        if ((h) && (h)->multi) {                                                           \
            if ((h)->multi->shard.size() != 1)                                             \
                return set_err(BT_EINVAL, "%s: not available on a multi-GPU handle", __func__); \
            (h) = (h)->multi->shard[0];                                                    \
        }                                                                                  \
    } while (0)

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char* bt_last_error(void) { return g_err.c_str(); }
const char* bt_version(void) { return "b200tally 0.1 (sm_100a)"; }

bt_status bt_create(const double* vertices, int64_t num_vertices, const int32_t* elements,
                    const int32_t* adj_elem, const int8_t* adj_face, int64_t num_elements,
                    const double* bbox, const double* centroid0, int64_t num_particles,
                    int32_t num_groups, int32_t device, bt_tally** out) {
    if (!out) return set_err(BT_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_particles <= 0) return set_err(BT_EINVAL, "num_particles must be positive");
    if (num_groups <= 0) return set_err(BT_EINVAL, "grid sizes must be positive");
    if (num_elements <= 0) return set_err(BT_EINVAL, "grid sizes must be positive");
    if (num_elements >= (1ll << 29)) return set_err(BT_EINVAL, "mesh too large (>= 2^29 tets)");
    if (num_particles >= (1ll << 31)) return set_err(BT_EINVAL, "capacity must be < 2^31");
    if (num_elements * (int64_t)num_groups >= (1ll << 40))
        return set_err(BT_EINVAL, "tally too large");
    if (!vertices || !elements || !adj_elem || !adj_face || !bbox || !centroid0)
        return set_err(BT_EINVAL, "NULL mesh array");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_err(BT_EINVAL, "device %d out of range (%d visible)", device, ndev);

    bt_tally* h = new bt_tally();
    h->dev = device;
    h->nv = num_vertices;
    h->ne = num_elements;
    h->cap = num_particles;
    h->ngroups = num_groups;
    memcpy(h->bbox, bbox, sizeof h->bbox);
    memcpy(h->c0, centroid0, sizeof h->c0);
    auto fail = [&](bt_status s) {
        std::string keep = g_err;
        free_all(h);
        delete h;
        g_err = keep;
        return s;
    };
    bt_status s = ensure_device(h);
    if (s) return fail(s);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(set_err(BT_ECUDA, "cudaGetDeviceProperties"));
    h->num_sms = prop.multiProcessorCount;
#define CKF(call)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(set_err(e_ == cudaErrorMemoryAllocation ? BT_ENOMEM : BT_ECUDA,  \
                                "%s failed: %s", #call, cudaGetErrorString(e_)));        \
    } while (0)
#define TRYF(x)                        \
    do {                               \
        bt_status s__ = (x);           \
        if (s__ != BT_OK) return fail(s__); \
    } while (0)
    CKF(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CKF(cudaEventCreate(&h->ev0));
    CKF(cudaEventCreate(&h->ev1));
    CKF(cudaEventCreate(&h->ev2));
    CKF(cudaEventCreate(&h->ev3));
    CKF(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    CKF(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
    {
        // localization of parked chunks at the highest priority: the walk's
        // persistent CTAs hold the SMs, a launch from this stream gets the
        // SMs freed between walk chunks first
        int lo_p = 0, hi_p = 0;
        CKF(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
        CKF(cudaStreamCreateWithPriority(&h->lstream, cudaStreamNonBlocking, hi_p));
    }
    CKF(cudaEventCreateWithFlags(&h->ev_s1, cudaEventDisableTiming));
    CKF(cudaEventCreateWithFlags(&h->ev_s2, cudaEventDisableTiming));
    CKF(cudaEventCreateWithFlags(&h->evc0, cudaEventDisableTiming));
    CKF(cudaEventCreateWithFlags(&h->evc1, cudaEventDisableTiming));
    CKF(cudaEventCreateWithFlags(&h->ev_loc, cudaEventDisableTiming));
    for (cudaEvent_t& e : h->evchunk) CKF(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CKF(cudaEventRecord(h->ev_loc, h->stream));

    // ---- mesh records (host packing, one upload)
    {
        std::vector<ElemRec> hr((size_t)num_elements);
        for (int64_t e = 0; e < num_elements; ++e) {
            for (int j = 0; j < 4; ++j) {
                const int v = elements[4 * e + j];
                if (v < 0 || v >= num_vertices)
                    return fail(set_err(BT_EINVAL, "element vertex id out of range"));
                hr[e].v[j] = v;
                const int nb = adj_elem[4 * e + j];
                const int nf = adj_face[4 * e + j];
                if (nb >= num_elements || (nb >= 0 && (nf < 0 || nf > 3)))
                    return fail(set_err(BT_EINVAL, "adjacency out of range"));
                hr[e].nb[j] = nb < 0 ? -1 : ((nb << 2) | nf);
            }
        }
        std::vector<Vtx> hv((size_t)num_vertices);
        for (int64_t v = 0; v < num_vertices; ++v)
            hv[v] = Vtx{vertices[3 * v], vertices[3 * v + 1], vertices[3 * v + 2], 0.0};
        TRYF(dalloc(&h->rec, num_elements));
        TRYF(dalloc(&h->vtx, num_vertices));
        CKF(cudaMemcpy(h->rec, hr.data(), sizeof(ElemRec) * hr.size(), cudaMemcpyHostToDevice));
        CKF(cudaMemcpy(h->vtx, hv.data(), sizeof(Vtx) * hv.size(), cudaMemcpyHostToDevice));
        TRYF(dalloc(&h->xrec, num_elements));
        // packed records need vertex ids < 2^24; B200TALLY_WIDE_XREC=1 forces the
        // wide layout on any mesh (tests)
        const char* wide_env = getenv("B200TALLY_WIDE_XREC");
        if (num_vertices >= (1 << 24) || (wide_env && atoi(wide_env) != 0))
            TRYF(dalloc(&h->xsel, num_elements));
        unsigned long long* dbad = nullptr;
        TRYF(dalloc(&dbad, 1));
        CKF(cudaMemset(dbad, 0, sizeof(unsigned long long)));
        xrec_kernel<<<grid_for(num_elements, 256), 256>>>(h->rec, num_elements, h->xrec, h->xsel, dbad);
        unsigned long long bad = 0;
        CKF(cudaMemcpy(&bad, dbad, sizeof(bad), cudaMemcpyDeviceToHost));
        cudaFree(dbad);
        if (bad) return fail(set_err(BT_EINVAL, "adjacency: a neighbour does not share the face's vertices"));
    }
    // ---- particles / staging / tallies
    const int64_t n = num_particles;
    TRYF(dalloc(&h->pos, 3 * n));
    TRYF(dalloc(&h->element, n));
    TRYF(dalloc(&h->alive, n));
    TRYF(dalloc(&h->entry, n));
    TRYF(dalloc(&h->stuck, n));
    TRYF(dalloc(&h->outcome, n));
    TRYF(dalloc(&h->seg_total, n));
    TRYF(dalloc(&h->group, n));
    TRYF(dalloc(&h->dest, 3 * n));
    TRYF(dalloc(&h->fly, n));
    TRYF(dalloc(&h->weight, n));
    const int64_t nbins = num_elements * num_groups;
    TRYF(dalloc(&h->tally, nbins));
    TRYF(dalloc(&h->sum, nbins));
    TRYF(dalloc(&h->sum_sq, nbins));
    TRYF(dalloc(&h->dcounters, NDCOUNTERS));
    CKF(cudaMallocHost((void**)&h->hcounters, NDCOUNTERS * sizeof(unsigned long long)));
    CKF(cudaMemset(h->pos, 0, sizeof(double) * 3 * n));
    CKF(cudaMemset(h->element, 0xff, sizeof(int32_t) * n));  // -1: unlocalized
    CKF(cudaMemset(h->alive, 0, n));
    CKF(cudaMemset(h->entry, 0xff, n));  // -1
    CKF(cudaMemset(h->stuck, 0, n));
    CKF(cudaMemset(h->outcome, 0, n));
    CKF(cudaMemset(h->seg_total, 0, sizeof(double) * n));
    CKF(cudaMemset(h->group, 0, sizeof(int32_t) * n));
    CKF(cudaMemset(h->tally, 0, sizeof(double) * nbins));
    CKF(cudaMemset(h->sum, 0, sizeof(double) * nbins));
    CKF(cudaMemset(h->sum_sq, 0, sizeof(double) * nbins));
    TRYF(build_grid(h));
    CKF(cudaStreamSynchronize(h->stream));
    *out = h;
    return BT_OK;
#undef CKF
#undef TRYF
}

bt_status bt_create_multi(const double* vertices, int64_t num_vertices, const int32_t* elements,
                          const int32_t* adj_elem, const int8_t* adj_face, int64_t num_elements,
                          const double* bbox, const double* centroid0, int64_t num_particles,
                          int32_t num_groups, const int32_t* devices, int32_t num_devices,
                          bt_tally** out) {
    if (!out) return set_err(BT_EINVAL, "out is NULL");
    *out = nullptr;
    if (!devices || num_devices <= 0) return set_err(BT_EINVAL, "need at least one device");
    if (num_particles <= 0) return set_err(BT_EINVAL, "num_particles must be positive");
    if (num_particles < num_devices)
        return set_err(BT_EINVAL, "num_particles (%lld) < number of devices (%d)",
                       (long long)num_particles, num_devices);
    return multi_create(vertices, num_vertices, elements, adj_elem, adj_face, num_elements, bbox,
                        centroid0, num_particles, num_groups, devices, num_devices, out);
}

bt_status bt_num_shards(bt_tally* h, int32_t* n) {
    if (!h || !n) return set_err(BT_EINVAL, "NULL argument");
    *n = h->multi ? (int32_t)h->multi->shard.size() : 1;
    return BT_OK;
}

bt_status bt_shard(bt_tally* h, int32_t index, bt_tally** shard, int64_t* lo, int64_t* hi) {
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (!h->multi) {
        if (index != 0) return set_err(BT_EINVAL, "shard index out of range");
        if (shard) *shard = h;
        if (lo) *lo = 0;
        if (hi) *hi = h->cap;
        return BT_OK;
    }
    if (index < 0 || index >= (int32_t)h->multi->shard.size())
        return set_err(BT_EINVAL, "shard index out of range");
    if (shard) *shard = h->multi->shard[(size_t)index];
    if (lo) *lo = h->multi->lo[(size_t)index];
    if (hi) *hi = h->multi->hi[(size_t)index];
    return BT_OK;
}

bt_status bt_destroy(bt_tally* h) {
    if (h && h->multi) {
        destroy_multi(h->multi);
        delete h;
        return BT_OK;
    }
    if (!h) return BT_OK;
    cudaSetDevice(h->dev);
    cudaStreamSynchronize(h->stream);
    cudaStreamSynchronize(h->cstream);
    if (h->lstream) cudaStreamSynchronize(h->lstream);
    free_all(h);
    delete h;
    return BT_OK;
}

bt_status bt_set_option(bt_tally* h, int32_t key, int64_t value) {
    if (h && h->multi) {
        Multi* m = h->multi;
        return fan_out(m, [&](int r) { return bt_set_option(m->shard[(size_t)r], key, value); });
    }
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    switch (key) {
        case BT_OPT_MAX_SWEEPS: h->max_sweeps = value; break;
        case BT_OPT_DIGEST:
            h->opt_digest = value != 0;
            if (h->opt_digest && !h->digest) {
                TRY(ensure_device(h));
                TRY(dalloc(&h->digest, h->cap));
                TRY(dalloc(&h->dcount, h->cap));
                CK(cudaMemset(h->dcount, 0, sizeof(int64_t) * h->cap));
            }
            break;
        case BT_OPT_SORT:
            h->opt_sort = value != 0;
            if (h->opt_sort && !h->order) {
                TRY(ensure_device(h));
                TRY(dalloc(&h->order, h->cap));
                TRY(dalloc(&h->sort_keys_in, h->cap));
                TRY(dalloc(&h->sort_keys_out, h->cap));
                TRY(dalloc(&h->sort_vals_in, h->cap));
                size_t b = 0;
                CK(cub::DeviceRadixSort::SortPairs(nullptr, b, h->sort_keys_in, h->sort_keys_out,
                                                   h->sort_vals_in, h->order, (int)h->cap));
                CK(cudaMalloc(&h->sort_tmp, b));
                h->sort_tmp_bytes = b;
            }
            break;
        case BT_OPT_WARP_AGG:
            if (value < 0 || value > 2)
                return set_err(BT_EINVAL, "warp aggregation must be 0 (adaptive), 1 or 2");
            h->opt_wagg = (int)value;
            break;
        case BT_OPT_BLOCKS_PER_SM: h->blocks_per_sm = (int)value; break;
        case BT_OPT_STAGED:
            if (value < 0 || value > 2)
                return set_err(BT_EINVAL, "staged must be 0 (v1), 1 (stage kernel) or 2 (direct)");
            h->opt_staged = (int)value;
            break;
        case BT_OPT_MOVE_CHUNKS: h->move_chunks = (int)value; break;
        case BT_OPT_EXACT_ONLY: h->opt_exact_only = value != 0; break;
        case BT_OPT_DEFER_INIT: h->opt_no_defer = value == 0; break;
        case BT_OPT_STREAM_MOVE: h->opt_stream_move = value != 0; break;
        case BT_OPT_LOCATE_LANES:
            if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8 &&
                value != 16 && value != 32)
                return set_err(BT_EINVAL, "locate lanes must be 0, 1, 2, 4, 8, 16 or 32");
            h->locate_lanes = (int)value;
            break;
        default: return set_err(BT_EINVAL, "unknown option %d", key);
    }
    return BT_OK;
}

static bt_status ensure_work(bt_tally* h) {
    if (h->work_mem) return BT_OK;
    const size_t n = (size_t)h->cap;
    char* p = nullptr;
    CK(cudaMalloc((void**)&p, n * (8 * sizeof(double) + sizeof(int4) + 4 * sizeof(int)) + 256));
    h->work_mem = p;
    WorkSoA& W = h->work;
    double* d = reinterpret_cast<double*>(p);
    W.px = d; W.py = d + n; W.pz = d + 2 * n; W.dx = d + 3 * n; W.dy = d + 4 * n;
    W.dz = d + 5 * n; W.w = d + 6 * n; W.seg = d + 7 * n;
    int4* r = reinterpret_cast<int4*>(d + 8 * n);
    W.r0 = r;
    int* q = reinterpret_cast<int*>(r + n);
    W.idx = q; W.e = q + n; W.g = q + 2 * n; W.fl = q + 3 * n;
    return BT_OK;
}

// Host work overlapped with the walk kernel (runs after the launch, before
// the stream synchronisation).
struct HostOverlap {
    void (*fn)(void*) = nullptr;
    void* ctx = nullptr;
};

static const struct Variant {
    int threads;
    void (*plain)(const WalkArgs);
    // [direct][digest]: direct refill or the stage kernel's work list; digests on/off
    void (*staged[2][2])(const WalkArgs, const WorkSoA, const int64_t*, const DirectArgs);
} kVariants[] = {
    // launch variant (CTA size, resident CTAs per SM = register budget);
    // BT_OPT_BLOCKS_PER_SM selects it, 0 = the tuned default
    {256, walk_kernel<256, 1>,
     {{walk_staged_kernel<256, 1, false, false>, walk_staged_kernel<256, 1, true, false>},
      {walk_staged_kernel<256, 1, false, true>, walk_staged_kernel<256, 1, true, true>}}},  // 1: <=255 regs
    {256, walk_kernel<256, 2>,
     {{walk_staged_kernel<256, 2, false, false>, walk_staged_kernel<256, 2, true, false>},
      {walk_staged_kernel<256, 2, false, true>, walk_staged_kernel<256, 2, true, true>}}},  // 2: <=128 regs
    {256, walk_kernel<256, 3>,
     {{walk_staged_kernel<256, 3, false, false>, walk_staged_kernel<256, 3, true, false>},
      {walk_staged_kernel<256, 3, false, true>, walk_staged_kernel<256, 3, true, true>}}},  // 3: <=80 regs
    {128, walk_kernel<128, 3>,
     {{walk_staged_kernel<128, 3, false, false>, walk_staged_kernel<128, 3, true, false>},
      {walk_staged_kernel<128, 3, false, true>, walk_staged_kernel<128, 3, true, true>}}},  // 4: <=168 regs
    {128, walk_kernel<128, 4>,
     {{walk_staged_kernel<128, 4, false, false>, walk_staged_kernel<128, 4, true, false>},
      {walk_staged_kernel<128, 4, false, true>, walk_staged_kernel<128, 4, true, true>}}},  // 5: <=128 regs
    {192, walk_kernel<192, 2>,
     {{walk_staged_kernel<192, 2, false, false>, walk_staged_kernel<192, 2, true, false>},
      {walk_staged_kernel<192, 2, false, true>, walk_staged_kernel<192, 2, true, true>}}},  // 6: <=168 regs
#ifdef BT_EXTRA_VARIANT  // experiments: -DBT_EXTRA_VARIANT -DBT_XV_T=224 -DBT_XV_B=2 -> variant 7
    {BT_XV_T, walk_kernel<BT_XV_T, BT_XV_B>,
     {{walk_staged_kernel<BT_XV_T, BT_XV_B, false, false>, walk_staged_kernel<BT_XV_T, BT_XV_B, true, false>},
      {walk_staged_kernel<BT_XV_T, BT_XV_B, false, true>, walk_staged_kernel<BT_XV_T, BT_XV_B, true, true>}}},
#endif
};

static WalkArgs walk_args(bt_tally* h, const double* dest, const int8_t* fly, const double* w,
                          bool score) {
    WalkArgs a;
    a.rec = h->rec;
    a.vtx = h->vtx;
    a.xrec = h->xrec;
    a.xsel = h->xsel;
    a.pos = h->pos;
    a.dest = dest;
    a.fly_in = fly;
    a.weight = w;
    a.group = h->group;
    a.element = h->element;
    a.alive = h->alive;
    a.entry = h->entry;
    a.stuck = h->stuck;
    a.outcome = h->outcome;
    a.seg_total = h->seg_total;
    a.tally = h->tally;
    const bool dig = h->opt_digest && score;
    a.digest = dig ? h->digest : nullptr;
    a.dcount = dig ? h->dcount : nullptr;
    a.order = nullptr;
    a.queue = h->dcounters + 16;
    a.counters = h->dcounters + 1;
    a.count = 0;
    a.max_sweeps = h->max_sweeps >= 0 ? h->max_sweeps : 2 * h->ne + 1000;
    a.max_sweeps32 = (int32_t)std::min<int64_t>(a.max_sweeps, 0x7fffffff);
    a.ngroups = h->ngroups;
    a.score = score ? 1 : 0;
    a.wagg = h->opt_wagg;
    a.exact_only = h->opt_exact_only ? 1 : 0;
    a.gate = nullptr;
    a.gate_pick = 0;
    a.ready = nullptr;
    return a;
}

// zero the move's counters; the first walk launch records ev0
static bt_status walk_begin(bt_tally* h) {
    CK(cudaMemsetAsync(h->dcounters, 0, sizeof(unsigned long long) * NDCOUNTERS, h->stream));
    h->walk_first = true;
    return BT_OK;
}

// one walk launch (+ its stage kernel / sort) of particles [lo, lo + count)
static bt_status launch_walk(bt_tally* h, WalkArgs a, int64_t lo, int64_t count, int chunk,
                             cudaStream_t st, bool direct) {
    const bool staged = h->opt_staged != 0;
    if (h->opt_sort && a.score) {  // whole move only (lo == 0)
        iota_keys_kernel<<<grid_for(count, 256), 256, 0, st>>>(
            h->element, count, h->sort_keys_in, h->sort_vals_in);
        CK(cudaGetLastError());
        size_t b = h->sort_tmp_bytes;
        CK(cub::DeviceRadixSort::SortPairs(h->sort_tmp, b, h->sort_keys_in, h->sort_keys_out,
                                           h->sort_vals_in, h->order, (int)count, 0, 32,
                                           st));
        a.order = h->order;
        h->kernels += 5;
    }
    constexpr int NVAR = sizeof(kVariants) / sizeof(kVariants[0]);
    const int vi = (h->blocks_per_sm >= 1 && h->blocks_per_sm <= NVAR ? h->blocks_per_sm
                                                                       : DEFAULT_VARIANT) - 1;
    const Variant& V = kVariants[vi];
    auto* staged_k = V.staged[direct ? 1 : 0][a.digest ? 1 : 0];
    const void* kptr = staged ? (const void*)staged_k : (const void*)V.plain;
    const size_t dyn = staged ? sizeof(WarpStage) * (direct ? 1 : 2) * (V.threads / 32) : 0;
    // the attribute and the occupancy of a (kernel, shared size) pair are
    // fixed: resolved on first use, then cached (two driver calls per launch
    // less: ~10 us of a 0.6-ms move of 1e5 particles)
    int bps = 0;
    for (const auto& c : h->occ)
        if (c.k == kptr && c.dyn == dyn) bps = c.bps;
    if (!bps) {
        if (staged)
            CK(cudaFuncSetAttribute(kptr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kptr, V.threads, dyn));
        bps = std::max(1, bps);
        h->occ.push_back({kptr, dyn, bps});
    }
    const int64_t want = (count + V.threads - 1) / V.threads;
    const unsigned blocks =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)bps * h->num_sms));
    int64_t* nwork = reinterpret_cast<int64_t*>(h->dcounters + 32 + chunk);
    WorkSoA W = h->work;
    DirectArgs D{lo, lo + count};
    if (direct && a.order) D = DirectArgs{0, count};  // sorted: slots index h->order
    if (staged && !direct) {
        TRY(ensure_work(h));
        W = h->work;
        W.px += lo; W.py += lo; W.pz += lo; W.dx += lo; W.dy += lo; W.dz += lo;
        W.r0 += lo;
        W.w += lo; W.seg += lo; W.idx += lo; W.e += lo; W.g += lo; W.fl += lo;
        stage_kernel<<<std::min<int64_t>(grid_for(count, 256), 16 * h->num_sms), 256, 0, st>>>(
            a, W, nwork, lo);
        CK(cudaGetLastError());
        h->kernels += 1;
    }
    if (h->walk_first) {
        CK(cudaEventRecord(h->ev0, st));
        h->walk_first = false;
    }
    if (staged)
        staged_k<<<blocks, V.threads, dyn, st>>>(a, W, nwork, D);
    else
        V.plain<<<blocks, V.threads, 0, st>>>(a);
    CK(cudaGetLastError());
    h->kernels += 1;
    return BT_OK;
}


// enqueue stage + walk of particles [lo, hi) as chunk `chunk` (staged path),
// or the whole range with the v1 kernel / element-sorted hand-out.
// pick_refill (single-launch moves): direct refill straight from the particle
// arrays, unless fewer than half the slots walk (chained moves after most
// particles leaked), where compacting first (stage kernel) wins -- decided on
// the device (WalkArgs::gate): both are enqueued, the other returns at once.
static bt_status walk_enqueue(bt_tally* h, WalkArgs a, int64_t lo, int64_t hi, int chunk,
                              cudaStream_t st = nullptr, bool pick_refill = false) {
    if (!st) st = h->stream;
    const int64_t count = hi - lo;
    a.count = count;
    a.queue = h->dcounters + 16 + chunk;
    // element-sorted hand-out: the stage kernel (direct gathers would be random)
    bool direct = h->opt_staged == 2 && !(h->opt_sort && a.score);
    if (direct && pick_refill && count >= (1 << 16)) {
        count_walkable_kernel<<<std::min<int64_t>(grid_for(count, 256), 1184), 256, 0, st>>>(
            a.fly_in + lo, h->element + lo, count, h->dcounters + 14);
        CK(cudaGetLastError());
        h->kernels += 1;
        a.gate = h->dcounters + 14;
        a.gate_pick = 1;
        TRY(launch_walk(h, a, lo, count, chunk, st, false));
        TRY(launch_walk(h, a, lo, count, chunk, st, true));
        return BT_OK;
    }
    return launch_walk(h, a, lo, count, chunk, st, direct);
}

// read the counters (running `overlap` on the host meanwhile) and fill the summary
static bt_status walk_end(bt_tally* h, int64_t max_sweeps, bt_summary* summary,
                          HostOverlap overlap = HostOverlap()) {
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaMemcpyAsync(h->hcounters, h->dcounters, sizeof(unsigned long long) * NDCOUNTERS,
                       cudaMemcpyDeviceToHost, h->stream));
    if (overlap.fn) overlap.fn(overlap.ctx);
    CK(cudaStreamSynchronize(h->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->walk_ms += ms;
    const unsigned long long* c = h->hcounters + 1;
    if (summary) {
        summary->sweeps = (int64_t)c[C_SWEEPS];
        summary->events = (int64_t)c[C_EVENTS];
        summary->reached = (int64_t)c[C_REACHED];
        summary->boundary_exits = (int64_t)c[C_BOUNDARY];
        summary->stuck_recoveries = (int64_t)c[C_RECOV];
        summary->stuck_terminations = (int64_t)c[C_KILLED];
    }
    if (c[C_ERR] & 2ull)
        return set_err(BT_ERUNTIME, "streamed move: inputs did not arrive within 5 s "
                                    "(BT_OPT_STREAM_MOVE = 0 walks chunk by chunk)");
    if (c[C_ERR])
        return set_err(BT_ERUNTIME, "trace did not terminate within %lld sweeps",
                       (long long)max_sweeps);
    if (c[C_UNLOC])
        return set_err(BT_EINVAL,
                       "%llu flying particle(s) not localized (element = -1) were not moved; "
                       "call initialize_particle_location first",
                       (unsigned long long)c[C_UNLOC]);
    return BT_OK;
}

static bt_status run_walk(bt_tally* h, const double* dest, const int8_t* fly, const double* w,
                          int64_t count, bool score, bt_summary* summary,
                          HostOverlap overlap = HostOverlap()) {
    WalkArgs a = walk_args(h, dest, fly, w, score);
    TRY(walk_begin(h));
    TRY(walk_enqueue(h, a, 0, count, 0, nullptr));
    return walk_end(h, a.max_sweeps, summary, overlap);
}

// lanes per particle of the grid search (BT_OPT_LOCATE_LANES; 0 = default)
constexpr int DEFAULT_LOCATE_LANES = 2;  // measured best on C2 and the 10M-tet cube (tools/locate_sweep.py)
static bt_status launch_locate(bt_tally* h, const LocateArgs& la, int64_t n,
                               cudaStream_t st = nullptr) {
    if (!st) st = h->stream;
    const int g = h->locate_lanes > 0 ? h->locate_lanes : DEFAULT_LOCATE_LANES;
    const int64_t threads = n * g;
    const unsigned blocks = (unsigned)((threads + LOCATE_THREADS - 1) / LOCATE_THREADS);
    switch (g) {
        case 1: locate_grid_kernel<1><<<blocks, LOCATE_THREADS, 0, st>>>(la); break;
        case 2: locate_grid_kernel<2><<<blocks, LOCATE_THREADS, 0, st>>>(la); break;
        case 4: locate_grid_kernel<4><<<blocks, LOCATE_THREADS, 0, st>>>(la); break;
        case 8: locate_grid_kernel<8><<<blocks, LOCATE_THREADS, 0, st>>>(la); break;
        case 16: locate_grid_kernel<16><<<blocks, LOCATE_THREADS, 0, st>>>(la); break;
        case 32: locate_grid_kernel<32><<<blocks, LOCATE_THREADS, 0, st>>>(la); break;
        default: return set_err(BT_EINVAL, "locate lanes must be 1, 2, 4, 8, 16 or 32");
    }
    CK(cudaGetLastError());
    h->kernels += 1;
    return BT_OK;
}

static LocateArgs locate_args(bt_tally* h, const double* target, int64_t count) {
    LocateArgs a;
    a.rec = h->rec;
    a.vtx = h->vtx;
    a.lam = h->lam;
    a.G = h->grid;
    a.target = target;
    a.pos = h->pos;
    a.element = h->element;
    a.alive = h->alive;
    a.entry = h->entry;
    a.stuck = h->stuck;
    a.outcome = h->outcome;
    a.seg_total = h->seg_total;
    memcpy(a.bbox, h->bbox, sizeof a.bbox);
    memcpy(a.c0, h->c0, sizeof a.c0);
    a.count = count;
    a.lo = 0;
    a.exact_only = h->opt_exact_only ? 1 : 0;
    return a;
}


// ---- deferred localization of host positions (see bt_tally::di_*)

// copy chunk k of the pending initialize from pos_stage and localize it
static bt_status di_enqueue(bt_tally* h, int k) {
    if (h->di_state[(size_t)k] != 1) return BT_OK;
    const int64_t lo = (int64_t)k * h->di_chunk, hi = std::min(h->di_count, lo + h->di_chunk);
    CK(cudaMemcpyAsync(h->init_stage + 3 * lo, h->pos_stage + 3 * lo,
                       sizeof(double) * 3 * (hi - lo), cudaMemcpyHostToDevice, h->cstream));
    CK(cudaEventRecord(h->di_cev[(size_t)k], h->cstream));
    CK(cudaStreamWaitEvent(h->lstream, h->di_cev[(size_t)k], 0));
    LocateArgs la = locate_args(h, h->init_stage, hi);
    la.lo = lo;
    TRY(launch_locate(h, la, hi - lo, h->lstream));
    CK(cudaEventRecord(h->di_ev[(size_t)k], h->lstream));
    h->di_state[(size_t)k] = 0;
    return BT_OK;
}

// stream `st` waits until particles [lo, hi) of the pending initialize are
// localized (enqueuing the parked chunks among them first)
static bt_status di_depend(bt_tally* h, int64_t lo, int64_t hi, cudaStream_t st) {
    if (!h->di_pending) return BT_OK;
    hi = std::min(hi, h->di_count);
    if (lo >= hi) return BT_OK;
    const int k0 = (int)(lo / h->di_chunk), k1 = (int)((hi - 1) / h->di_chunk);
    for (int k = k0; k <= k1; ++k) {
        TRY(di_enqueue(h, k));
        CK(cudaStreamWaitEvent(st, h->di_ev[(size_t)k], 0));
    }
    return BT_OK;
}

// finish the pending initialize: every parked chunk copied and localized,
// the main stream ordered after all of it
static bt_status settle_init(bt_tally* h) {
    if (!h->di_pending) return BT_OK;
    for (int k = 0; k < h->di_nch; ++k) TRY(di_enqueue(h, k));
    CK(cudaEventRecord(h->ev_loc, h->lstream));
    CK(cudaStreamWaitEvent(h->stream, h->ev_loc, 0));
    h->di_pending = false;
    return BT_OK;
}

// initialize_particle_location with host positions, grid mode, count >=
// DEFER_MIN: the caller's buffer is consumed from both ends at once -- the
// DMA engine copies chunks from the front straight out of a pinned buffer
// (each localized as soon as it lands), host threads copy chunks from the
// back into the pinned pos_stage -- and the call returns when they meet
// (PCIe + host memcpy bandwidth, ~90 GB/s on the GPU box instead of the DMA's
// 53: tools/micro/hostcopy.cu).  The parked chunks are copied and localized
// by the next move, interleaved with its own input copies, right before the
// walk chunks that need them.  A pageable buffer is all parked.
// Opt-in (BT_OPT_DEFER_INIT = 1): the call returns 1.3 ms sooner (C2, 1e7
// pinned positions: 3.1 vs 4.5 ms), but the parked half's localization then
// runs while the move's persistent walk CTAs hold every SM, so it waits for
// a walk chunk to drain and the walk chunk after it waits for it: the move
// takes 2.4 ms longer (tools/e2e_breakdown.py, profiles/r02_e2e_breakdown.txt).
constexpr int64_t DEFER_MIN = 1 << 20;
constexpr int64_t DI_CHUNK_BYTES = 8 << 20;
static bt_status init_host_deferred(bt_tally* h, const double* positions, int64_t count,
                                    bool pageable) {
    if (!h->init_stage) TRY(dalloc(&h->init_stage, 3 * h->cap));
    if (!h->pos_stage) CK(cudaMallocHost((void**)&h->pos_stage, sizeof(double) * 3 * h->cap));
    if (!h->stager) h->stager = new HostStager();
    TRY(h->stager->init());
    // the previous localization (and its reads of init_stage) is complete
    CK(cudaStreamWaitEvent(h->cstream, h->ev_loc, 0));
    CK(cudaStreamWaitEvent(h->lstream, h->ev_loc, 0));
    const int64_t P = std::max<int64_t>(1, DI_CHUNK_BYTES / 24);
    const int nch = (int)((count + P - 1) / P);
    h->di_count = count;
    h->di_chunk = P;
    h->di_nch = nch;
    h->di_state.assign((size_t)nch, 0);
    while ((int)h->di_ev.size() < nch) {
        cudaEvent_t a, b;
        CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        h->di_ev.push_back(a);
        h->di_cev.push_back(b);
    }
    std::mutex mu;
    int front = 0, back = nch - 1;  // next chunk for the DMA / for the host threads
    int last_dma = -1;
    bt_status st_dma = BT_OK;
    std::string err_dma;
    HostPool* pool = h->stager->pool;
    pool->run([&](int i) {
        if (i == 0 && !pageable) {  // the calling thread feeds the DMA engine
            std::vector<int> inflight;
            for (;;) {
                int k;
                {
                    std::lock_guard<std::mutex> g(mu);
                    if (front > back) break;
                    k = front++;
                }
                const int64_t lo = (int64_t)k * P, hi = std::min(count, lo + P);
                cudaError_t e = cudaMemcpyAsync(h->init_stage + 3 * lo, positions + 3 * lo,
                                                sizeof(double) * 3 * (hi - lo),
                                                cudaMemcpyHostToDevice, h->cstream);
                if (e == cudaSuccess) e = cudaEventRecord(h->di_cev[(size_t)k], h->cstream);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(h->lstream, h->di_cev[(size_t)k], 0);
                if (e != cudaSuccess) {
                    st_dma = set_err(BT_ECUDA, "deferred initialize: %s", cudaGetErrorString(e));
                    err_dma = g_err;
                    std::lock_guard<std::mutex> g(mu);
                    front = back + 1;
                    break;
                }
                LocateArgs la = locate_args(h, h->init_stage, hi);
                la.lo = lo;
                const bt_status ls = launch_locate(h, la, hi - lo, h->lstream);
                if (ls != BT_OK || cudaEventRecord(h->di_ev[(size_t)k], h->lstream) != cudaSuccess) {
                    st_dma = ls != BT_OK ? ls : set_err(BT_ECUDA, "deferred initialize: event");
                    err_dma = g_err;
                    std::lock_guard<std::mutex> g(mu);
                    front = back + 1;
                    break;
                }
                last_dma = k;
                // keep two copies queued: enough to keep the engine busy, few
                // enough that the meeting point follows the actual rates
                inflight.push_back(k);
                if (inflight.size() > 2) {
                    cudaEventSynchronize(h->di_cev[(size_t)inflight.front()]);
                    inflight.erase(inflight.begin());
                }
            }
            return;
        }
        for (;;) {  // host threads park chunks from the back
            int k;
            {
                std::lock_guard<std::mutex> g(mu);
                if (back < front) break;
                k = back--;
            }
            const int64_t lo = (int64_t)k * P, hi = std::min(count, lo + P);
            memcpy(h->pos_stage + 3 * lo, positions + 3 * lo, sizeof(double) * 3 * (hi - lo));
            h->di_state[(size_t)k] = 1;
        }
    });
    if (st_dma != BT_OK) {
        g_err = err_dma;
        return st_dma;
    }
    // the caller's buffer must be read before returning: the last front copy
    if (last_dma >= 0) CK(cudaEventSynchronize(h->di_cev[(size_t)last_dma]));
    h->di_pending = true;
    return BT_OK;
}

bt_status bt_initialize_particle_location(bt_tally* h, const double* positions, int64_t size,
                                          int32_t mem_kind, int32_t mode, bt_summary* summary) {
    if (h && h->multi) return multi_initialize(h, positions, size, mem_kind, mode, summary);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (summary) memset(summary, 0, sizeof *summary);
    if (size < 0 || size % 3 != 0)
        return set_err(BT_EINVAL, "positions must hold 3*count floats, got %lld",
                       (long long)size);
    const int64_t count = size / 3;
    if (count > h->cap)
        return set_err(BT_EINVAL, "count %lld exceeds capacity %lld", (long long)count,
                       (long long)h->cap);
    if (mode != BT_LOCATE_GRID && mode != BT_LOCATE_WALK)
        return set_err(BT_EINVAL, "unknown localization mode %d", mode);
    TRY(ensure_device(h));
    h->walk_ms = 0.f;
    h->kernels = 0;
    h->source_weight = 0.0;
    if (count == 0) return BT_OK;
    if (!positions) return set_err(BT_EINVAL, "positions is NULL");
    CK(cudaEventRecord(h->ev2, h->stream));
    const double* target = positions;
    const bool host = mem_kind == BT_MEM_HOST;
    TRY(settle_init(h));  // a previous initialize's parked chunks
    if (host && mode == BT_LOCATE_GRID && count >= DEFER_MIN && !h->opt_no_defer) {
        TRY(init_host_deferred(h, positions, count, is_pageable(positions)));
        CK(cudaEventRecord(h->ev3, h->stream));
        h->call_pending = true;
        return BT_OK;
    }
    if (host && mode == BT_LOCATE_GRID) {
        // Copy on the copy stream into a dedicated staging buffer, then
        // return as soon as the caller's buffer has been read: the
        // localization kernel runs on while the next call's copies proceed
        // (every later kernel or readout is ordered after it on `stream`).
        // Chunked: chunk c's localization starts as soon as its positions
        // have landed, while the next chunks are still being copied.
        if (!h->init_stage) TRY(dalloc(&h->init_stage, 3 * h->cap));
        CK(cudaStreamWaitEvent(h->cstream, h->ev_loc, 0));  // previous localization done
        int nch_big = 4;
        if (const char* env = getenv("B200TALLY_INIT_CHUNKS")) nch_big = std::max(1, std::min(MAX_CHUNKS, atoi(env)));
        const int nch = (int)std::min<int64_t>(count >= (4 << 20) ? nch_big : 1, count);
        const bool pageable = is_pageable(positions);
        LocateArgs la = locate_args(h, h->init_stage, count);
        for (int c = 0; c < nch; ++c) {
            const int64_t lo = count * c / nch, hi = count * (c + 1) / nch;
            TRY(h2d(h, h->init_stage + 3 * lo, positions + 3 * lo,
                    sizeof(double) * 3 * (hi - lo), h->cstream, pageable));
            CK(cudaEventRecord(h->evchunk[c], h->cstream));
            CK(cudaStreamWaitEvent(h->stream, h->evchunk[c], 0));
            la.lo = lo;
            la.count = hi;
            TRY(launch_locate(h, la, hi - lo));
        }
        CK(cudaEventRecord(h->evc0, h->cstream));
        CK(cudaEventRecord(h->ev_loc, h->stream));
        CK(cudaEventRecord(h->ev3, h->stream));
        // a pinned caller buffer is read by the DMA engine: wait for it; a
        // pageable one has already been copied into the library's ring
        if (!pageable) CK(cudaEventSynchronize(h->evc0));
        h->call_pending = true;
        return BT_OK;
    }
    if (host) {
        TRY(h2d(h, h->dest, positions, sizeof(double) * 3 * count, h->stream,
                is_pageable(positions)));
        target = h->dest;
    }
    LocateArgs la = locate_args(h, target, count);
    if (mode == BT_LOCATE_GRID) {
        TRY(launch_locate(h, la, count));
    } else {
        init_walk_prep_kernel<<<grid_for(count, 256), 256, 0, h->stream>>>(la, h->fly);
        CK(cudaGetLastError());
        h->kernels += 1;
        TRY(run_walk(h, target, h->fly, nullptr, count, false, summary));
        tiebreak_kernel<<<grid_for(count, 128), 128, 0, h->stream>>>(la);
        CK(cudaGetLastError());
        h->kernels += 1;
    }
    CK(cudaEventRecord(h->ev_loc, h->stream));
    CK(cudaEventRecord(h->ev3, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaEventElapsedTime(&h->call_ms, h->ev2, h->ev3));
    h->call_pending = false;
    return BT_OK;
}

// The recorded source weight of a device-input move, on the device: the
// flying particles' weights compacted in index order, then numpy's pairwise
// summation tree (move_prep.cuh) into dcounters[DC_SOURCE_WEIGHT] -- the
// same bits as the host-input path and the reference (tally.py:267-269).
static bt_status device_source_weight(bt_tally* h, const int8_t* flying, const double* weights,
                                      int64_t count, cudaStream_t st) {
    if (!h->wsel) {
        int depth = 0;
        while ((h->cap >> depth) > 64) ++depth;
        h->wsel_depth = depth;
        TRY(dalloc(&h->wsel, h->cap));
        TRY(dalloc(&h->wsel_vals, (int64_t)2 << depth));
        TRY(dalloc(&h->wsel_ticks, (int64_t)2 << depth));
        CK(cudaMemset(h->wsel_ticks, 0, sizeof(unsigned) * ((size_t)2 << depth)));
        size_t b = 0;
        CK(cub::DeviceSelect::Flagged(nullptr, b, weights, flying, h->wsel,
                                      reinterpret_cast<long long*>(h->dcounters + DC_SELECTED),
                                      (int)h->cap));
        CK(cudaMalloc(&h->wsel_tmp, b));
        h->wsel_tmp_bytes = b;
    }
    size_t b = h->wsel_tmp_bytes;
    long long* m = reinterpret_cast<long long*>(h->dcounters + DC_SELECTED);
    CK(cub::DeviceSelect::Flagged(h->wsel_tmp, b, weights, flying, h->wsel, m, (int)count, st));
    const int64_t nthreads = (int64_t)1 << h->wsel_depth;
    pairwise_sum_kernel<<<grid_for(nthreads, 256), 256, 0, st>>>(
        h->wsel, m, h->wsel_depth, h->wsel_vals, h->wsel_ticks,
        reinterpret_cast<double*>(h->dcounters + DC_SOURCE_WEIGHT));
    CK(cudaGetLastError());
    h->kernels += 3;
    return BT_OK;
}

bt_status bt_move_to_next_location(bt_tally* h, const double* destinations, const int8_t* flying,
                                   const double* weights, const int32_t* groups, int64_t size,
                                   int32_t mem_kind, bt_summary* summary) {
    if (h && h->multi)
        return multi_move(h, destinations, flying, weights, groups, size, mem_kind, summary);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (summary) memset(summary, 0, sizeof *summary);
    const int64_t count = size;
    if (count < 0 || count > h->cap)
        return set_err(BT_EINVAL, "count %lld outside [0, %lld]", (long long)count,
                       (long long)h->cap);
    TRY(ensure_device(h));
    h->walk_ms = 0.f;
    h->kernels = 0;
    if (count == 0) return BT_OK;
    if (!destinations || !flying || !weights)
        return set_err(BT_EINVAL, "NULL move array");
    const bool host = mem_kind == BT_MEM_HOST;
    // host-side checks and the recorded source weight (tally.py:262-269)
    bool need_w = h->source_weight == 0.0;
    if (host) {
        if (groups) {  // range check before any work, in parallel blocks
            const int64_t bad = first_bad_group(groups, count, h->ngroups);
            if (bad >= 0)
                return set_err(BT_EINDEX, "group %d out of range [0, %d)", groups[bad],
                               h->ngroups);
        }
    }
    CK(cudaEventRecord(h->ev2, h->stream));
    // the recorded source weight (host inputs: numpy's pairwise order, computed
    // on the host while the walk kernels run; device inputs: summed in stage)
    struct WJob {
        const double* w;
        const int8_t* fly;
        int64_t n;
        double* sel;  // persistent host scratch (no page faults per call)
        double out;
    } job{weights, flying, count, nullptr, 0.0};
    HostOverlap ov;
    if (host && need_w) {
        if ((int64_t)h->host_sel.size() < count) h->host_sel.assign((size_t)h->cap, 0.0);
        job.sel = h->host_sel.data();
        ov.ctx = &job;
        ov.fn = [](void* c) {
            WJob* j = static_cast<WJob*>(c);
            const int nt = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
            const int64_t m = select_flying(j->w, j->fly, j->n, j->sel, nt);
            j->out = m < 0 ? pairwise_sum_par(j->w, j->n, 3) : pairwise_sum_par(j->sel, m, 3);
        };
    }
    bt_status s;
    if (host) {
        // pipeline: chunk c's input copies (copy stream) overlap chunk c-1's walk.
        // Chunks grow geometrically (1/2^nch, then 1/2^(nch-1-c) cumulative:
        // 1/16, 3/16, 1/4, 1/2 for the default four: measured best of 2..6 chunks,
        // tools/e2e_breakdown.py) so the first walk starts after a short copy
        // and every later copy still finishes inside the previous chunk's walk.
        WalkArgs a = walk_args(h, h->dest, h->fly, h->weight, true);
        int nch = 1;
        if (h->opt_staged && !h->opt_sort) {
            nch = h->move_chunks > 0 ? h->move_chunks : (count >= (4 << 20) ? 4 : 1);
            nch = (int)std::min<int64_t>(std::min(nch, MAX_CHUNKS), count);
        }
        // Streamed: one direct-refill launch over the whole move; its warps wait
        // for each chunk's inputs (WalkArgs::ready) instead of one launch per
        // chunk, whose tails cost ~1 ms of the C2 move.  Chunk ends are
        // multiples of 128 particles, so no L1 line of a landed chunk holds
        // bytes of one still in flight.
        const bool any_pageable = is_pageable(destinations) || is_pageable(flying) ||
                                  is_pageable(weights) || (groups && is_pageable(groups));
        // Pinned (or registered) inputs only: every copy and mark is enqueued
        // before the walk is launched, so nothing the walk waits for depends on
        // the host after the launch -- a tool that runs the launch alone (ncu)
        // or to completion (CUDA_LAUNCH_BLOCKING) cannot deadlock it.
        // Pageable inputs are staged by host threads while the walk runs and
        // keep one launch per chunk.
        // (From 2^18 particles: below that the copies are a few tens of us.)
        bool streamed = h->opt_stream_move && h->opt_staged == 2 && !h->opt_sort &&
                        !h->di_pending && !any_pageable &&
                        (h->move_chunks > 1 || (h->move_chunks <= 0 && count >= (1 << 18)));
        if (streamed && h->stream_ops != 0) {
            if (!h->ready) TRY(dalloc(&h->ready, 1));
            streamed = stream_write(h, h->ready, 0, h->cstream);
            if (h->stream_ops < 0) h->stream_ops = streamed ? 1 : 0;
            if (!streamed) cudaGetLastError();
        } else {
            streamed = false;
        }
        // Streamed marks: the walk starts after 1/64 of the inputs and the
        // copies (~1600 particles/us pinned) outrun the walk (~700/us on C2)
        // from there, so the marks only need to come often: 1/64, 1/32,
        // 1/16, 1/8, then every 1/8 (or move_chunks equal parts if set).
        static const double kMarks[] = {1 / 64., 1 / 32., 1 / 16., 1 / 8., 2 / 8., 3 / 8.,
                                        4 / 8.,  5 / 8.,  6 / 8.,  7 / 8., 1.0};
        if (streamed && h->move_chunks <= 0) nch = (int)(sizeof kMarks / sizeof kMarks[0]);
        auto bound = [&](int c) -> int64_t {  // end of chunk c
            if (c + 1 >= nch) return count;
            if (streamed) {
                const double f = h->move_chunks > 0 ? (double)(c + 1) / nch : kMarks[c];
                return (int64_t)((double)count * f) & ~(int64_t)127;
            }
            const int sh = c == 0 ? nch : nch - 1 - c;
            return (int64_t)((double)count / (double)(1ll << sh));
        };
        const bool pg_dest = is_pageable(destinations), pg_fly = is_pageable(flying),
                   pg_w = is_pageable(weights), pg_g = groups && is_pageable(groups);
        TRY(walk_begin(h));
        // odd chunks go to a second stream, so chunk c+1's CTAs take the SMs
        // that chunk c's tail frees instead of waiting for its last walk
        CK(cudaEventRecord(h->ev_s1, h->stream));
        CK(cudaStreamWaitEvent(h->stream2, h->ev_s1, 0));
        if (streamed) {
            for (int c = 0; c < nch; ++c) {
                const int64_t lo = c == 0 ? 0 : bound(c - 1), hi = bound(c);
                const int64_t n = hi - lo;  // (the first chunk may round to empty)
                TRY(h2d(h, h->dest + 3 * lo, destinations + 3 * lo, sizeof(double) * 3 * n,
                        h->cstream, pg_dest));
                TRY(h2d(h, h->fly + lo, flying + lo, n, h->cstream, pg_fly));
                TRY(h2d(h, h->weight + lo, weights + lo, sizeof(double) * n, h->cstream, pg_w));
                if (groups)
                    TRY(h2d(h, h->group + lo, groups + lo, sizeof(int32_t) * n, h->cstream, pg_g));
                if (!stream_write(h, h->ready, (unsigned long long)hi, h->cstream))
                    return set_err(BT_ECUDA, "stream memory write failed");
                if (c == 0) {  // the walk starts once the first chunk has landed
                    CK(cudaEventRecord(h->evchunk[0], h->cstream));
                    CK(cudaStreamWaitEvent(h->stream, h->evchunk[0], 0));
                }
            }
            WalkArgs sa = a;
            sa.ready = h->ready;
            TRY(walk_enqueue(h, sa, 0, count, 0, h->stream));
            // the move ends after the copy stream's last write
            CK(cudaEventRecord(h->evchunk[1], h->cstream));
            CK(cudaStreamWaitEvent(h->stream, h->evchunk[1], 0));
        }
        for (int c = 0; c < (streamed ? 0 : nch); ++c) {
            const int64_t lo = c == 0 ? 0 : bound(c - 1), hi = bound(c);
            const int64_t n = hi - lo;
            if (n <= 0) continue;
            cudaStream_t st = (c & 1) ? h->stream2 : h->stream;
            // the pending initialize's chunks under [lo, hi): copied and
            // localized now, ahead of this chunk's own inputs
            TRY(di_depend(h, lo, hi, st));
            TRY(h2d(h, h->dest + 3 * lo, destinations + 3 * lo, sizeof(double) * 3 * n,
                    h->cstream, pg_dest));
            TRY(h2d(h, h->fly + lo, flying + lo, n, h->cstream, pg_fly));
            TRY(h2d(h, h->weight + lo, weights + lo, sizeof(double) * n, h->cstream, pg_w));
            if (groups)
                TRY(h2d(h, h->group + lo, groups + lo, sizeof(int32_t) * n, h->cstream, pg_g));
            CK(cudaEventRecord(h->evchunk[c], h->cstream));
            CK(cudaStreamWaitEvent(st, h->evchunk[c], 0));
            TRY(walk_enqueue(h, a, lo, hi, c, st));
        }
        CK(cudaEventRecord(h->ev_s2, h->stream2));
        CK(cudaStreamWaitEvent(h->stream, h->ev_s2, 0));
        TRY(settle_init(h));  // particles beyond this move's count
        s = walk_end(h, a.max_sweeps, summary, ov);
        if (need_w) h->source_weight = job.out;
    } else {
        // Device inputs: one host synchronisation per move.  The group range
        // check, the refill choice and the recorded source weight are all
        // decided on the device, and come back with the counters in one copy.
        TRY(settle_init(h));
        WalkArgs a = walk_args(h, destinations, flying, weights, true);
        TRY(walk_begin(h));
        a.gate = h->dcounters + 14;  // [14] walkable, [15] prepare_kernel's flags
        if (groups) {
            CK(cudaMemcpyAsync(h->group, groups, sizeof(int32_t) * count,
                               cudaMemcpyDeviceToDevice, h->stream));
            prepare_kernel<<<grid_for(count, 256), 256, 0, h->stream>>>(
                flying, h->element, h->group, h->ngroups, count, h->dcounters + 15);
            CK(cudaGetLastError());
            h->kernels += 1;
        }
        if (need_w) {  // on the second stream: overlaps the walk (its tail, at least)
            CK(cudaEventRecord(h->ev_s1, h->stream));
            CK(cudaStreamWaitEvent(h->stream2, h->ev_s1, 0));
            TRY(device_source_weight(h, flying, weights, count, h->stream2));
            CK(cudaEventRecord(h->ev_s2, h->stream2));
        }
        TRY(walk_enqueue(h, a, 0, count, 0, nullptr, true));
        if (need_w) CK(cudaStreamWaitEvent(h->stream, h->ev_s2, 0));
        s = walk_end(h, a.max_sweeps, summary);
        if (h->hcounters[15] & 2ull)
            return set_err(BT_EINDEX, "group out of range [0, %d)", h->ngroups);
        if (need_w && s == BT_OK) {
            double dw;
            memcpy(&dw, h->hcounters + DC_SOURCE_WEIGHT, sizeof dw);
            h->source_weight = dw;
        }
    }
    CK(cudaEventRecord(h->ev3, h->stream));
    CK(cudaEventSynchronize(h->ev3));
    CK(cudaEventElapsedTime(&h->call_ms, h->ev2, h->ev3));
    h->call_pending = false;
    return s;
}

bt_status bt_finalize_batch(bt_tally* h, double source_weight) {
    if (h && h->multi) return multi_finalize(h, source_weight);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    double w = source_weight > 0.0 ? source_weight : h->source_weight;
    if (!(w > 0.0))
        return set_err(BT_ERUNTIME, "no source weight recorded for this batch; pass source_weight");
    TRY(ensure_device(h));
    const int64_t nb = h->ne * h->ngroups;
    finalize_kernel<<<grid_for(nb, 256), 256, 0, h->stream>>>(h->tally, h->sum, h->sum_sq, nb, w);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    h->batches += 1;
    h->source_weight = 0.0;
    return BT_OK;
}

static double* tally_ptr(bt_tally* h, int32_t which) {
    switch (which) {
        case BT_TALLY_BATCH: return h->tally;
        case BT_TALLY_SUM: return h->sum;
        case BT_TALLY_SUM_SQ: return h->sum_sq;
        case BT_TALLY_COL_BATCH: return h->col_tally;
        case BT_TALLY_COL_SUM: return h->col_sum;
        case BT_TALLY_COL_SUM_SQ: return h->col_sum_sq;
        default: return nullptr;
    }
}

bt_status bt_read_tally(bt_tally* h, int32_t which, double* out, int64_t n) {
    if (h && h->multi) return multi_read_tally(h, which, out, n);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    double* p = tally_ptr(h, which);
    if (!p) return set_err(BT_EINVAL, "unknown tally array %d", which);
    if (n != h->ne * h->ngroups) return set_err(BT_EINVAL, "n must be E*G");
    TRY(ensure_device(h));
    CK(cudaMemcpyAsync(out, p, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return BT_OK;
}

bt_status bt_tally_device_ptr(bt_tally* h, int32_t which, void** ptr) {
    MULTI_SINGLE(h);
    if (!h || !ptr) return set_err(BT_EINVAL, "NULL argument");
    double* p = tally_ptr(h, which);
    if (!p) return set_err(BT_EINVAL, "unknown tally array %d", which);
    // a consumer on another stream must see every kernel enqueued so far
    TRY(ensure_device(h));
    CK(cudaStreamSynchronize(h->stream));
    *ptr = p;
    return BT_OK;
}

bt_status bt_get_source_weight(bt_tally* h, double* w) {
    if (h && h->multi && w) {
        *w = h->multi->source_weight;
        return BT_OK;
    }
    if (!h || !w) return set_err(BT_EINVAL, "NULL argument");
    *w = h->source_weight;
    return BT_OK;
}

bt_status bt_set_source_weight(bt_tally* h, double w) {
    if (h && h->multi) {
        h->multi->source_weight = w;
        for (bt_tally* t : h->multi->shard) t->source_weight = w;
        return BT_OK;
    }
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    h->source_weight = w;
    return BT_OK;
}

bt_status bt_batches_completed(bt_tally* h, int64_t* n) {
    if (h && h->multi) h = h->multi->shard[0];
    if (!h || !n) return set_err(BT_EINVAL, "NULL argument");
    *n = h->batches;
    return BT_OK;
}

bt_status bt_read_particles(bt_tally* h, int64_t count, double* position, int32_t* element,
                            int8_t* alive, int8_t* entry_face, int8_t* stuck, int8_t* outcome,
                            double* seg_total) {
    if (h && h->multi)
        return multi_read_particles(h, count, position, element, alive, entry_face, stuck, outcome,
                                    seg_total);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (count < 0 || count > h->cap) return set_err(BT_EINVAL, "count out of range");
    TRY(ensure_device(h));
    TRY(settle_init(h));
    auto cp = [&](void* dst, const void* src, size_t bytes) -> bt_status {
        if (dst && bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
        return BT_OK;
    };
    TRY(cp(position, h->pos, sizeof(double) * 3 * count));
    TRY(cp(element, h->element, sizeof(int32_t) * count));
    TRY(cp(alive, h->alive, count));
    TRY(cp(entry_face, h->entry, count));
    TRY(cp(stuck, h->stuck, count));
    TRY(cp(outcome, h->outcome, count));
    TRY(cp(seg_total, h->seg_total, sizeof(double) * count));
    CK(cudaStreamSynchronize(h->stream));
    return BT_OK;
}

bt_status bt_read_digest(bt_tally* h, int64_t count, uint64_t* digest, int64_t* events) {
    if (h && h->multi) return multi_read_digest(h, count, digest, events);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (!h->digest) return set_err(BT_EINVAL, "digests are off (BT_OPT_DIGEST)");
    if (count < 0 || count > h->cap) return set_err(BT_EINVAL, "count out of range");
    TRY(ensure_device(h));
    TRY(settle_init(h));
    if (digest)
        CK(cudaMemcpyAsync(digest, h->digest, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost,
                           h->stream));
    if (events)
        CK(cudaMemcpyAsync(events, h->dcount, sizeof(int64_t) * count, cudaMemcpyDeviceToHost,
                           h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return BT_OK;
}

bt_status bt_last_timing(bt_tally* h, float* walk_ms, float* call_ms, int64_t* kernels) {
    if (h && h->multi) return multi_last_timing(h, walk_ms, call_ms, kernels);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (h->call_pending) {
        TRY(ensure_device(h));
        CK(cudaEventSynchronize(h->ev3));
        CK(cudaEventElapsedTime(&h->call_ms, h->ev2, h->ev3));
        h->call_pending = false;
    }
    if (walk_ms) *walk_ms = h->walk_ms;
    if (call_ms) *call_ms = h->call_ms;
    if (kernels) *kernels = h->kernels;
    return BT_OK;
}

bt_status bt_particle_device_ptrs(bt_tally* h, double** position, int32_t** element,
                                  int8_t** alive) {
    MULTI_SINGLE(h);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    // the localization of host positions completes asynchronously: a consumer
    // on another stream (e.g. torch's) must see its element / pos / alive
    TRY(ensure_device(h));
    TRY(settle_init(h));
    CK(cudaStreamSynchronize(h->stream));
    if (position) *position = h->pos;
    if (element) *element = h->element;
    if (alive) *alive = h->alive;
    return BT_OK;
}

bt_status bt_save_state(bt_tally* h) {
    if (h && h->multi) {
        Multi* m = h->multi;
        return fan_out(m, [&](int r) { return bt_save_state(m->shard[(size_t)r]); });
    }
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    TRY(ensure_device(h));
    TRY(settle_init(h));
    const int64_t n = h->cap;
    if (!h->snap_pos) {
        TRY(dalloc(&h->snap_pos, 3 * n));
        TRY(dalloc(&h->snap_element, n));
        TRY(dalloc(&h->snap_flags, 4 * n));
        TRY(dalloc(&h->snap_seg, n));
    }
    auto d2d = cudaMemcpyDeviceToDevice;
    CK(cudaMemcpyAsync(h->snap_pos, h->pos, sizeof(double) * 3 * n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->snap_element, h->element, sizeof(int32_t) * n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->snap_flags, h->alive, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->snap_flags + n, h->entry, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->snap_flags + 2 * n, h->stuck, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->snap_flags + 3 * n, h->outcome, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->snap_seg, h->seg_total, sizeof(double) * n, d2d, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->have_snapshot = true;
    return BT_OK;
}

bt_status bt_restore_state(bt_tally* h) {
    if (h && h->multi) {
        Multi* m = h->multi;
        return fan_out(m, [&](int r) { return bt_restore_state(m->shard[(size_t)r]); });
    }
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (!h->have_snapshot) return set_err(BT_EINVAL, "no snapshot saved");
    TRY(ensure_device(h));
    TRY(settle_init(h));
    const int64_t n = h->cap;
    auto d2d = cudaMemcpyDeviceToDevice;
    CK(cudaMemcpyAsync(h->pos, h->snap_pos, sizeof(double) * 3 * n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->element, h->snap_element, sizeof(int32_t) * n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->alive, h->snap_flags, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->entry, h->snap_flags + n, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->stuck, h->snap_flags + 2 * n, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->outcome, h->snap_flags + 3 * n, n, d2d, h->stream));
    CK(cudaMemcpyAsync(h->seg_total, h->snap_seg, sizeof(double) * n, d2d, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return BT_OK;
}

bt_status bt_build_adjacency(const int32_t* elements, int64_t num_elements, int64_t num_vertices,
                             int32_t device, int32_t* adj_elem, int8_t* adj_face) {
    if (num_elements < 0 || num_vertices < 0) return set_err(BT_EINVAL, "negative sizes");
    if (num_elements >= (1ll << 29)) return set_err(BT_EINVAL, "mesh too large (>= 2^29 tets)");
    if (num_elements == 0) return BT_OK;
    if (!elements || !adj_elem || !adj_face) return set_err(BT_EINVAL, "NULL array");
    for (int64_t i = 0; i < 4 * num_elements; ++i)
        if (elements[i] < 0 || elements[i] >= num_vertices)
            return set_err(BT_EINVAL, "element vertex id out of range");
    CK(cudaSetDevice(device));
    const int64_t ne = num_elements, nrows = 4 * ne;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int *d_el = nullptr, *rows = nullptr, *rows2 = nullptr, *ae = nullptr;
    unsigned *kc = nullptr, *kc2 = nullptr, *flags = nullptr;
    unsigned long long *kab = nullptr, *kab2 = nullptr;
    signed char* af = nullptr;
    long long* err = nullptr;
    void* tmp = nullptr;
    bt_status rc = BT_OK;
    auto cleanup = [&]() {
        void* ps[] = {d_el, rows, rows2, ae, kc, kc2, flags, kab, kab2, af, err, tmp};
        for (void* p : ps)
            if (p) cudaFree(p);
        cudaStreamDestroy(st);
    };
#define CKA(call)                                                                       \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            rc = set_err(e_ == cudaErrorMemoryAllocation ? BT_ENOMEM : BT_ECUDA,        \
                         "%s failed: %s", #call, cudaGetErrorString(e_));               \
            cleanup();                                                                  \
            return rc;                                                                  \
        }                                                                               \
    } while (0)
    CKA(cudaMalloc(&d_el, sizeof(int) * nrows));
    CKA(cudaMalloc(&rows, sizeof(int) * nrows));
    CKA(cudaMalloc(&rows2, sizeof(int) * nrows));
    CKA(cudaMalloc(&kc, sizeof(unsigned) * nrows));
    CKA(cudaMalloc(&kc2, sizeof(unsigned) * nrows));
    CKA(cudaMalloc(&kab, sizeof(unsigned long long) * nrows));
    CKA(cudaMalloc(&kab2, sizeof(unsigned long long) * nrows));
    CKA(cudaMalloc(&ae, sizeof(int) * nrows));
    CKA(cudaMalloc(&af, nrows));
    CKA(cudaMalloc(&flags, sizeof(unsigned)));
    CKA(cudaMalloc(&err, 3 * sizeof(long long)));
    CKA(cudaMemcpyAsync(d_el, elements, sizeof(int) * nrows, cudaMemcpyHostToDevice, st));
    CKA(cudaMemsetAsync(ae, 0xff, sizeof(int) * nrows, st));
    CKA(cudaMemsetAsync(af, 0xff, nrows, st));
    CKA(cudaMemsetAsync(flags, 0, sizeof(unsigned), st));
    CKA(cudaMemsetAsync(err, 0x7f, 3 * sizeof(long long), st));
    int vbits = 1;
    while ((1ll << vbits) < num_vertices + 1) ++vbits;
    adj_keys_c_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(d_el, nrows, kc, rows);
    CKA(cudaGetLastError());
    size_t b1 = 0, b2 = 0;
    CKA(cub::DeviceRadixSort::SortPairs(nullptr, b1, kc, kc2, rows, rows2, (int)nrows, 0, vbits, st));
    CKA(cub::DeviceRadixSort::SortPairs(nullptr, b2, kab, kab2, rows2, rows, (int)nrows, 0,
                                        32 + vbits, st));
    CKA(cudaMalloc(&tmp, std::max(b1, b2)));
    CKA(cub::DeviceRadixSort::SortPairs(tmp, b1, kc, kc2, rows, rows2, (int)nrows, 0, vbits, st));
    adj_keys_ab_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(d_el, nrows, rows2, kab);
    CKA(cudaGetLastError());
    CKA(cub::DeviceRadixSort::SortPairs(tmp, b2, kab, kab2, rows2, rows, (int)nrows, 0, 32 + vbits,
                                        st));
    adj_match_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(d_el, nrows, rows, ae, af, flags, err);
    CKA(cudaGetLastError());
    adj_dup_kernel<<<grid_for(ne, 256), 256, 0, st>>>(ae, ne, flags, err);
    CKA(cudaGetLastError());
    unsigned hflags = 0;
    long long herr[3];
    CKA(cudaMemcpyAsync(&hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, st));
    CKA(cudaMemcpyAsync(herr, err, sizeof herr, cudaMemcpyDeviceToHost, st));
    CKA(cudaMemcpyAsync(adj_elem, ae, sizeof(int) * nrows, cudaMemcpyDeviceToHost, st));
    CKA(cudaMemcpyAsync(adj_face, af, nrows, cudaMemcpyDeviceToHost, st));
    CKA(cudaStreamSynchronize(st));
    if (hflags & 1u) {
        int row = 0;
        CKA(cudaMemcpy(&row, rows + herr[0], sizeof row, cudaMemcpyDeviceToHost));
        const int64_t e = row >> 2, f = row & 3;
        int v[3], j = 0;
        for (int q = 0; q < 4; ++q)
            if (q != f) v[j++] = elements[4 * e + q];
        std::sort(v, v + 3);
        rc = set_err(BT_EINVAL,
                     "face with vertices (%d, %d, %d) is shared by more than two elements "
                     "(duplicate or non-manifold mesh)", v[0], v[1], v[2]);
    } else if (hflags & 2u) {
        rc = set_err(BT_EINVAL, "element %lld lists the same face twice (repeated vertex id)",
                     herr[1]);
    } else if (hflags & 4u) {
        rc = set_err(BT_EINVAL, "element %lld duplicates element %d", herr[2],
                     adj_elem[4 * herr[2]]);
    }
    cleanup();
#undef CKA
    return rc;
}

bt_status bt_transport_run(bt_tally* h, const double* sigma_t, const double* sigma_s_row_prob,
                           const double* group_cdf, int32_t num_groups, int64_t num_particles,
                           int64_t num_batches, uint64_t seed, const double* box,
                           const double* fixed_direction, bt_transport_totals* out) {
    MULTI_SINGLE(h);
    if (!h || !sigma_t || !sigma_s_row_prob || !group_cdf || !box || !out)
        return set_err(BT_EINVAL, "NULL argument");
    if (num_groups != h->ngroups)
        return set_err(BT_EINVAL, "cross sections have %d groups, the tally %d", num_groups,
                       h->ngroups);
    if (num_particles <= 0 || num_particles > h->cap)
        return set_err(BT_EINVAL, "num_particles must be in [1, %lld]", (long long)h->cap);
    if (num_batches <= 0) return set_err(BT_EINVAL, "num_batches must be positive");
    memset(out, 0, sizeof *out);
    TRY(ensure_device(h));
    TRY(settle_init(h));
    const int64_t n = num_particles, nb = h->ne * h->ngroups, G = num_groups;
    if (!h->col_tally) {
        TRY(dalloc(&h->col_tally, nb));
        TRY(dalloc(&h->col_sum, nb));
        TRY(dalloc(&h->col_sum_sq, nb));
        CK(cudaMemset(h->col_tally, 0, sizeof(double) * nb));
        CK(cudaMemset(h->col_sum, 0, sizeof(double) * nb));
        CK(cudaMemset(h->col_sum_sq, 0, sizeof(double) * nb));
        TRY(dalloc(&h->tr_dir, 3 * h->cap));
        TRY(dalloc(&h->tr_weight, h->cap));
        TRY(dalloc(&h->tr_rng, h->cap));
        TRY(dalloc(&h->tr_round_max, MAX_ROUNDS_TRACKED));
        TRY(dalloc(&h->tr_count, 4));
        TRY(dalloc(&h->tr_wsum, 4));
        TRY(dalloc(&h->tr_xs, 2 * G + G * G));
    }
    if (!h->init_stage) TRY(dalloc(&h->init_stage, 3 * h->cap));
    CK(cudaMemcpyAsync(h->tr_xs, sigma_t, sizeof(double) * G, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->tr_xs + G, sigma_s_row_prob, sizeof(double) * G, cudaMemcpyHostToDevice,
                       h->stream));
    CK(cudaMemcpyAsync(h->tr_xs + 2 * G, group_cdf, sizeof(double) * G * G,
                       cudaMemcpyHostToDevice, h->stream));
    TransportArgs t;
    t.w = walk_args(h, nullptr, nullptr, nullptr, true);
    t.w.group = h->group;
    t.xs = XSDev{h->tr_xs, h->tr_xs + G, h->tr_xs + 2 * G, num_groups};
    t.col_tally = h->col_tally;
    t.dir = h->tr_dir;
    t.rng_block = h->tr_rng;
    t.group_rw = h->group;
    t.weight_rw = h->tr_weight;
    t.src = h->init_stage;
    t.round_max = h->tr_round_max;
    t.tcount = h->tr_count;
    t.wsum = h->tr_wsum;
    t.queue = h->dcounters + 16;
    t.seed = seed;
    t.n = n;
    t.max_rounds = 50000000;  // _MAX_ROUNDS, transport.py:296
    const int fixed = fixed_direction != nullptr;
    const double fdx = fixed ? fixed_direction[0] : 0.0, fdy = fixed ? fixed_direction[1] : 0.0,
                 fdz = fixed ? fixed_direction[2] : 0.0;
    // launch variant: BT_OPT_BLOCKS_PER_SM = 1 -> 256 threads x 1 CTA/SM (<= 255 registers),
    // otherwise 192 x 2 (<= 168 registers, the walk's default shape)
    const bool wide = h->blocks_per_sm == 1;
    const int tthreads = wide ? 256 : 192;
    const void* tk = wide ? (const void*)transport_kernel<256, 1> : (const void*)transport_kernel<192, 2>;
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, tk, tthreads, 0));
    bps = std::max(1, bps);
    const unsigned blocks = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((n + tthreads - 1) / tthreads, (int64_t)bps * h->num_sms));
    LocateArgs la = locate_args(h, h->init_stage, n);
    h->kernels = 0;
    float loc_ms = 0.f, batch_ms = 0.f;
    for (int64_t b = 0; b < num_batches; ++b) {
        t.batch = (uint64_t)b;
        CK(cudaMemsetAsync(h->dcounters, 0, sizeof(unsigned long long) * NDCOUNTERS, h->stream));
        CK(cudaMemsetAsync(h->tr_round_max, 0, sizeof(unsigned) * MAX_ROUNDS_TRACKED, h->stream));
        CK(cudaMemsetAsync(h->tr_count, 0, sizeof(unsigned long long) * 4, h->stream));
        CK(cudaMemsetAsync(h->tr_wsum, 0, sizeof(double) * 4, h->stream));
        CK(cudaEventRecord(h->ev2, h->stream));
        transport_source_kernel<<<grid_for(n, 256), 256, 0, h->stream>>>(
            t, box[0], box[1], box[2], box[3], box[4], box[5], fixed, fdx, fdy, fdz,
            h->init_stage);
        CK(cudaGetLastError());
        TRY(launch_locate(h, la, n));
        CK(cudaGetLastError());
        CK(cudaEventRecord(h->ev0, h->stream));
        count_alive_kernel<<<std::min<int64_t>(grid_for(n, 256), 1024), 256, 0, h->stream>>>(
            h->alive, n, h->tr_count + 2);
        if (wide)
            transport_kernel<256, 1><<<blocks, 256, 0, h->stream>>>(t);
        else
            transport_kernel<192, 2><<<blocks, 192, 0, h->stream>>>(t);
        CK(cudaGetLastError());
        sum_rounds_kernel<<<256, 256, 0, h->stream>>>(h->tr_round_max, MAX_ROUNDS_TRACKED,
                                                      h->tr_count + 1);
        seg_sum_kernel<<<std::min<int64_t>(grid_for(n, 256), 1024), 256, 0, h->stream>>>(
            h->seg_total, h->alive, n, h->tr_wsum + 3);
        CK(cudaGetLastError());
        CK(cudaEventRecord(h->ev1, h->stream));
        h->kernels += 6;
        unsigned long long cnt[4];
        double ws[4];
        CK(cudaMemcpyAsync(cnt, h->tr_count, sizeof cnt, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(ws, h->tr_wsum, sizeof ws, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(h->hcounters, h->dcounters, sizeof(unsigned long long) * NDCOUNTERS,
                           cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        float m1 = 0.f, m2 = 0.f;
        CK(cudaEventElapsedTime(&m1, h->ev2, h->ev0));
        CK(cudaEventElapsedTime(&m2, h->ev0, h->ev1));
        loc_ms += m1;
        batch_ms += m2;
        const unsigned long long* c = h->hcounters + 1;
        if (c[C_ERR]) return set_err(BT_ERUNTIME, "transport did not terminate");
        const double bsw = (double)cnt[2];  // sum of unit source weights of located particles
        if (!(bsw > 0.0)) return set_err(BT_ERUNTIME, "no source particle inside the mesh");
        out->source_weight += bsw;
        out->leaked_weight += ws[0];
        out->absorbed_weight += ws[1];
        out->stuck_weight += ws[2];
        out->track_length_total += ws[3];
        out->collisions += (int64_t)cnt[0];
        out->sweeps += (int64_t)cnt[1];
        out->events += (int64_t)c[C_EVENTS];
        const int64_t nbins = nb;
        finalize_kernel<<<grid_for(nbins, 256), 256, 0, h->stream>>>(h->tally, h->sum, h->sum_sq,
                                                                     nbins, bsw);
        finalize_kernel<<<grid_for(nbins, 256), 256, 0, h->stream>>>(
            h->col_tally, h->col_sum, h->col_sum_sq, nbins, bsw);
        CK(cudaGetLastError());
        h->kernels += 2;
        h->batches += 1;
        h->col_batches += 1;
    }
    CK(cudaStreamSynchronize(h->stream));
    out->ms_localization = loc_ms;
    out->ms_transport = batch_ms;
    h->walk_ms = batch_ms;
    h->source_weight = 0.0;
    return BT_OK;
}

bt_status bt_read_transport_state(bt_tally* h, int64_t count, double* direction, int32_t* group,
                                  uint32_t* rng_block) {
    MULTI_SINGLE(h);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (!h->tr_dir) return set_err(BT_EINVAL, "no transport run on this handle");
    if (count < 0 || count > h->cap) return set_err(BT_EINVAL, "count out of range");
    TRY(ensure_device(h));
    if (direction)
        CK(cudaMemcpyAsync(direction, h->tr_dir, sizeof(double) * 3 * count,
                           cudaMemcpyDeviceToHost, h->stream));
    if (group)
        CK(cudaMemcpyAsync(group, h->group, sizeof(int32_t) * count, cudaMemcpyDeviceToHost,
                           h->stream));
    if (rng_block)
        CK(cudaMemcpyAsync(rng_block, h->tr_rng, sizeof(uint32_t) * count,
                           cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return BT_OK;
}

bt_status bt_uniform_blocks(const uint64_t* keys, int64_t n, int32_t device, double* out) {
    if (n <= 0) return BT_OK;
    if (!keys || !out) return set_err(BT_EINVAL, "NULL argument");
    CK(cudaSetDevice(device));
    uint64_t* dk = nullptr;
    double* dout = nullptr;
    CK(cudaMalloc(&dk, sizeof(uint64_t) * 4 * n));
    CK(cudaMalloc(&dout, sizeof(double) * 4 * n));
    CK(cudaMemcpy(dk, keys, sizeof(uint64_t) * 4 * n, cudaMemcpyHostToDevice));
    philox_kat_kernel<<<grid_for(n, 128), 128>>>(dk, n, dout);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost);
    cudaFree(dk);
    cudaFree(dout);
    if (e != cudaSuccess) return set_err(BT_ECUDA, "philox: %s", cudaGetErrorString(e));
    return BT_OK;
}

__global__ void glibc_math_kernel(const double* __restrict__ x, int64_t n, int fn,
                                  double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
#if BT_GLIBC_MATH
    if (i >= n) return;
    out[i] = fn == 0 ? gm_log(x[i]) : fn == 1 ? gm_sin(x[i]) : gm_cos(x[i]);
#else
    if (i >= n) return;
    out[i] = fn == 0 ? log(x[i]) : fn == 1 ? sin(x[i]) : cos(x[i]);
#endif
}

bt_status bt_glibc_math(const double* x, int64_t n, int32_t fn, int32_t device, double* out) {
    if (!BT_GLIBC_MATH)
        return set_err(BT_EINVAL, "built without the host libm tables (BT_GLIBC_MATH 0)");
    if (fn < 0 || fn > 2) return set_err(BT_EINVAL, "fn must be 0 (log), 1 (sin) or 2 (cos)");
    if (n <= 0) return BT_OK;
    if (!x || !out) return set_err(BT_EINVAL, "NULL argument");
    CK(cudaSetDevice(device));
    double *dx = nullptr, *dout = nullptr;
    CK(cudaMalloc(&dx, sizeof(double) * n));
    CK(cudaMalloc(&dout, sizeof(double) * n));
    cudaError_t e = cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        glibc_math_kernel<<<grid_for(n, 256), 256>>>(dx, n, fn, dout);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dout);
    if (e != cudaSuccess) return set_err(BT_ECUDA, "glibc math: %s", cudaGetErrorString(e));
    return BT_OK;
}

static bt_status ensure_sweep_bufs(bt_tally* h) {
    if (h->sb_mem) return BT_OK;
    const size_t n = (size_t)h->cap;
    // 8-byte arrays first, then 4-byte, then 1-byte
    // 15 doubles/int64, 8 int32 (+1 for the scan total), 7 int8 per particle; 22
    // sub-arrays each rounded up to 256 bytes
    const size_t bytes = n * (8 * 15 + 4 * 8 + 7) + 4 + 22 * 256 + 256;
    char* p = nullptr;
    CK(cudaMalloc((void**)&p, bytes));
    h->sb_mem = p;
    SweepBufs& B = h->sb;
    auto take = [&](size_t b) { char* q = p; p += (b + 255) & ~size_t(255); return q; };
    B.s_start = (double*)take(8 * 3 * n);
    B.s_end = (double*)take(8 * 3 * n);
    B.s_len = (double*)take(8 * n);
    B.e_start = (double*)take(8 * 3 * n);
    B.e_end = (double*)take(8 * 3 * n);
    B.e_len = (double*)take(8 * n);
    B.e_particle = (int64_t*)take(8 * n);
    B.active = (int32_t*)take(4 * n);
    B.has_ev = (int32_t*)take(4 * n);
    B.offs = (int32_t*)take(4 * (n + 1));
    B.s_elem = (int32_t*)take(4 * n);
    B.s_next = (int32_t*)take(4 * n);
    B.e_elem = (int32_t*)take(4 * n);
    B.e_next = (int32_t*)take(4 * n);
    B.e_next_prop = (int32_t*)take(4 * n);
    B.s_face = (int8_t*)take(n);
    B.s_entry = (int8_t*)take(n);
    B.s_done = (int8_t*)take(n);
    B.e_face = (int8_t*)take(n);
    B.e_done = (int8_t*)take(n);
    B.e_entry = (int8_t*)take(n);
    B.e_done_prop = (int8_t*)take(n);
    TRY(dalloc(&h->sb_flag, h->cap + 1));
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, h->sb_flag, B.offs, (int)(h->cap + 1)));
    CK(cudaMalloc(&h->sb_tmp, tb));
    h->sb_tmp_bytes = tb;
    return BT_OK;
}

bt_status bt_load_step(bt_tally* h, const double* destinations, const int8_t* flying,
                       const double* weights, const int32_t* groups, int64_t count,
                       int32_t mem_kind) {
    MULTI_SINGLE(h);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (count < 0 || count > h->cap)
        return set_err(BT_EINVAL, "count %lld outside [0, %lld]", (long long)count,
                       (long long)h->cap);
    TRY(ensure_device(h));
    TRY(settle_init(h));
    if (count == 0) return BT_OK;
    if (!destinations || !flying || !weights) return set_err(BT_EINVAL, "NULL array");
    if (!h->tr_fly) TRY(dalloc(&h->tr_fly, h->cap));
    const cudaMemcpyKind kind = mem_kind == BT_MEM_HOST ? cudaMemcpyHostToDevice
                                                        : cudaMemcpyDeviceToDevice;
    if (groups && mem_kind == BT_MEM_HOST)
        for (int64_t i = 0; i < count; ++i)
            if (groups[i] < 0 || groups[i] >= h->ngroups)
                return set_err(BT_EINDEX, "group %d out of range [0, %d)", groups[i], h->ngroups);
    if (mem_kind == BT_MEM_HOST) {
        TRY(h2d(h, h->dest, destinations, sizeof(double) * 3 * count, h->stream,
                is_pageable(destinations)));
        TRY(h2d(h, h->fly, flying, count, h->stream, is_pageable(flying)));
        TRY(h2d(h, h->weight, weights, sizeof(double) * count, h->stream, is_pageable(weights)));
        if (groups)
            TRY(h2d(h, h->group, groups, sizeof(int32_t) * count, h->stream, is_pageable(groups)));
    } else {
        CK(cudaMemcpyAsync(h->dest, destinations, sizeof(double) * 3 * count, kind, h->stream));
        CK(cudaMemcpyAsync(h->fly, flying, count, kind, h->stream));
        CK(cudaMemcpyAsync(h->weight, weights, sizeof(double) * count, kind, h->stream));
        if (groups)
            CK(cudaMemcpyAsync(h->group, groups, sizeof(int32_t) * count, kind, h->stream));
    }
    load_step_kernel<<<grid_for(h->cap, 256), 256, 0, h->stream>>>(h->fly, count, h->cap,
                                                                    h->tr_fly, h->alive);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    h->loaded = count;
    return BT_OK;
}

__global__ void unlocalized_kernel(const int8_t* __restrict__ fly, const int32_t* __restrict__ el,
                                   int64_t n, unsigned long long* __restrict__ first) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && fly[i] && el[i] < 0) atomicMin(first, (unsigned long long)i);
}

bt_status bt_trace_begin(bt_tally* h, int32_t score, int64_t max_sweeps) {
    MULTI_SINGLE(h);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    TRY(ensure_device(h));
    TRY(settle_init(h));
    if (!h->tr_fly) return set_err(BT_EINVAL, "no step loaded (bt_load_step)");
    TRY(ensure_sweep_bufs(h));
    // _check_localized (search.py:440-446)
    CK(cudaMemsetAsync(h->dcounters + 15, 0xff, sizeof(unsigned long long), h->stream));
    unlocalized_kernel<<<grid_for(h->cap, 256), 256, 0, h->stream>>>(h->tr_fly, h->element,
                                                                      h->cap, h->dcounters + 15);
    unsigned long long first = 0;
    CK(cudaMemcpyAsync(&first, h->dcounters + 15, sizeof first, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (first != ~0ull)
        return set_err(BT_EINVAL,
                       "flying particle %llu is not localized (element = -1); call "
                       "initialize_locations first", first);
    CK(cudaMemsetAsync(h->dcounters, 0, sizeof(unsigned long long) * NDCOUNTERS, h->stream));
    if (h->opt_digest) {
        // fresh per-call digests (the recorder view of the test harness)
        fill_digest_kernel<<<grid_for(h->cap, 256), 256, 0, h->stream>>>(h->digest, h->dcount,
                                                                         h->cap);
        CK(cudaGetLastError());
    }
    h->tr_score = score != 0;
    h->tr_sweeps = 0;
    h->tr_events = 0;
    h->tr_nev = 0;
    h->tr_limit = max_sweeps >= 0 ? max_sweeps : 2 * h->ne + 1000;
    return BT_OK;
}

bt_status bt_trace_propose(bt_tally* h, bt_sweep_events* ev, int64_t* flying) {
    MULTI_SINGLE(h);
    if (!h || !ev || !flying) return set_err(BT_EINVAL, "NULL argument");
    TRY(ensure_device(h));
    const int64_t n = h->cap;
    SweepBufs& B = h->sb;
    // compact flying (ascending), search.py:160-166
    select_flying_kernel<<<grid_for(n, 256), 256, 0, h->stream>>>(h->tr_fly, n, h->sb_flag);
    CK(cudaMemsetAsync(h->sb_flag + n, 0, sizeof(int32_t), h->stream));
    size_t tb = h->sb_tmp_bytes;
    CK(cub::DeviceScan::ExclusiveSum(h->sb_tmp, tb, h->sb_flag, B.offs, (int)(n + 1), h->stream));
    scatter_active_kernel<<<grid_for(n, 256), 256, 0, h->stream>>>(h->sb_flag, B.offs, n,
                                                                    B.active);
    int32_t m32 = 0;
    CK(cudaMemcpyAsync(&m32, B.offs + n, sizeof m32, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const int64_t m = m32;
    *flying = m;
    memset(ev, 0, sizeof *ev);
    h->tr_nev = 0;
    if (m == 0) return BT_OK;
    WalkArgs a = walk_args(h, h->dest, h->tr_fly, h->weight, h->tr_score);
    sweep_propose_kernel<<<grid_for(m, 128), 128, 0, h->stream>>>(a, h->tr_fly, B, m);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(B.has_ev + m, 0, sizeof(int32_t), h->stream));
    tb = h->sb_tmp_bytes;
    CK(cub::DeviceScan::ExclusiveSum(h->sb_tmp, tb, B.has_ev, B.offs, (int)(m + 1), h->stream));
    sweep_compact_kernel<<<grid_for(m, 256), 256, 0, h->stream>>>(B, m);
    CK(cudaGetLastError());
    int32_t nev = 0;
    CK(cudaMemcpyAsync(&nev, B.offs + m, sizeof nev, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->tr_nev = nev;
    ev->count = nev;
    ev->particle = B.e_particle;
    ev->element = B.e_elem;
    ev->exit_face = B.e_face;
    ev->segment_start = B.e_start;
    ev->segment_end = B.e_end;
    ev->segment_length = B.e_len;
    ev->next_element = B.e_next;
    ev->particle_done = B.e_done;
    ev->next_proposed = B.e_next_prop;
    return BT_OK;
}

bt_status bt_trace_commit(bt_tally* h) {
    MULTI_SINGLE(h);
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    TRY(ensure_device(h));
    const int64_t nev = h->tr_nev;
    if (nev > 0) {
        WalkArgs a = walk_args(h, h->dest, h->tr_fly, h->weight, h->tr_score);
        a.digest = h->opt_digest ? h->digest : nullptr;
        a.dcount = h->opt_digest ? h->dcount : nullptr;
        sweep_commit_kernel<<<grid_for(nev, 256), 256, 0, h->stream>>>(a, h->tr_fly, h->sb, nev);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
    }
    h->tr_events += nev;
    h->tr_sweeps += 1;
    h->tr_nev = 0;
    if (h->tr_sweeps > h->tr_limit)
        return set_err(BT_ERUNTIME, "trace did not terminate within %lld sweeps",
                       (long long)h->tr_limit);
    return BT_OK;
}

bt_status bt_trace_end(bt_tally* h, bt_summary* out) {
    MULTI_SINGLE(h);
    if (!h || !out) return set_err(BT_EINVAL, "NULL argument");
    TRY(ensure_device(h));
    CK(cudaMemcpyAsync(h->hcounters, h->dcounters, sizeof(unsigned long long) * NDCOUNTERS,
                       cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const unsigned long long* c = h->hcounters + 1;
    out->sweeps = h->tr_sweeps;
    out->events = h->tr_events;
    out->reached = (int64_t)c[C_REACHED];
    out->boundary_exits = (int64_t)c[C_BOUNDARY];
    out->stuck_recoveries = (int64_t)c[C_RECOV];
    out->stuck_terminations = (int64_t)c[C_KILLED];
    return BT_OK;
}

bt_status bt_memcpy(void* dst, const void* src, int64_t bytes, int32_t kind) {
    if (bytes <= 0) return BT_OK;
    if (!dst || !src) return set_err(BT_EINVAL, "NULL pointer");
    CK(cudaMemcpy(dst, src, (size_t)bytes,
                  kind == 0 ? cudaMemcpyDeviceToHost
                            : (kind == 1 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice)));
    return BT_OK;
}

bt_status bt_flux(bt_tally* h, int32_t estimator, const double* volumes, double* mean,
                  double* rel_error) {
    if (h && h->multi) h = h->multi->shard[0];  // finalized moments: the same on every GPU
    if (!h || !volumes || !mean || !rel_error) return set_err(BT_EINVAL, "NULL argument");
    const double* sm = estimator == 0 ? h->sum : h->col_sum;
    const double* sq = estimator == 0 ? h->sum_sq : h->col_sum_sq;
    const int64_t n = estimator == 0 ? h->batches : h->col_batches;
    if (!sm) return set_err(BT_EINVAL, "no collision estimator on this handle");
    if (n == 0) return set_err(BT_ERUNTIME, "no batches completed; nothing to normalize");
    for (int64_t e = 0; e < h->ne; ++e)
        if (!(volumes[e] > 0.0)) return set_err(BT_EINVAL, "volumes must be positive");
    TRY(ensure_device(h));
    const int64_t nb = h->ne * h->ngroups;
    double *dv = nullptr, *dm = nullptr, *dr = nullptr;
    TRY(dalloc(&dv, h->ne));
    TRY(dalloc(&dm, nb));
    TRY(dalloc(&dr, nb));
    cudaError_t err = cudaMemcpyAsync(dv, volumes, sizeof(double) * h->ne, cudaMemcpyHostToDevice,
                                      h->stream);
    if (err == cudaSuccess) {
        flux_kernel<<<grid_for(nb, 256), 256, 0, h->stream>>>(sm, sq, dv, h->ne, h->ngroups, n, dm,
                                                              dr);
        err = cudaGetLastError();
    }
    if (err == cudaSuccess)
        err = cudaMemcpyAsync(mean, dm, sizeof(double) * nb, cudaMemcpyDeviceToHost, h->stream);
    if (err == cudaSuccess)
        err = cudaMemcpyAsync(rel_error, dr, sizeof(double) * nb, cudaMemcpyDeviceToHost,
                              h->stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize(h->stream);
    cudaFree(dv);
    cudaFree(dm);
    cudaFree(dr);
    if (err != cudaSuccess) return set_err(BT_ECUDA, "bt_flux: %s", cudaGetErrorString(err));
    return BT_OK;
}

bt_status bt_info(bt_tally* h, int32_t* device, int64_t* num_elements, int64_t* capacity,
                  int32_t* num_groups) {
    if (h && h->multi) {
        if (device) *device = h->multi->shard[0]->dev;
        if (num_elements) *num_elements = h->ne;
        if (capacity) *capacity = h->multi->cap;
        if (num_groups) *num_groups = h->ngroups;
        return BT_OK;
    }
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (device) *device = h->dev;
    if (num_elements) *num_elements = h->ne;
    if (capacity) *capacity = h->cap;
    if (num_groups) *num_groups = h->ngroups;
    return BT_OK;
}


// ---- standalone tally grids and scoring (tally.py:21-80)

bt_status bt_create_grid(int64_t num_elements, int32_t num_groups, int32_t device,
                         bt_tally** out) {
    if (!out) return set_err(BT_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_elements <= 0 || num_groups <= 0)
        return set_err(BT_EINVAL, "grid sizes must be positive, got (%lld, %d)",
                       (long long)num_elements, num_groups);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_err(BT_EINVAL, "device %d out of range (%d visible)", device, ndev);
    bt_tally* h = new bt_tally();
    h->dev = device;
    h->ne = num_elements;
    h->ngroups = num_groups;
    h->cap = 0;  // no particles: moves of count > 0 are refused
    auto fail = [&](bt_status st) {
        const std::string keep = g_err;
        free_all(h);
        delete h;
        g_err = keep;
        return st;
    };
    bt_status st = ensure_device(h);
    if (st) return fail(st);
    const int64_t nb = num_elements * num_groups;
    if ((st = dalloc(&h->tally, nb)) || (st = dalloc(&h->sum, nb)) || (st = dalloc(&h->sum_sq, nb)) ||
        (st = dalloc(&h->dcounters, NDCOUNTERS)))
        return fail(st);
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMemset(h->tally, 0, sizeof(double) * nb) != cudaSuccess ||
        cudaMemset(h->sum, 0, sizeof(double) * nb) != cudaSuccess ||
        cudaMemset(h->sum_sq, 0, sizeof(double) * nb) != cudaSuccess)
        return fail(set_err(BT_ECUDA, "bt_create_grid: %s", cudaGetErrorString(cudaGetLastError())));
    *out = h;
    return BT_OK;
}

bt_status bt_score(bt_tally* h, int32_t kind, const int32_t* elements, const int32_t* groups,
                   const double* weights, const double* values, int64_t n, int32_t mem_kind) {
    if (h && h->multi) h = h->multi->shard[0];  // BT_TALLY_BATCH is the sum over GPUs
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (kind != 0 && kind != 1) return set_err(BT_EINVAL, "kind must be 0 (track) or 1 (collision)");
    if (n < 0) return set_err(BT_EINVAL, "negative count");
    if (n == 0) return BT_OK;
    if (!elements || !groups || !weights || !values) return set_err(BT_EINVAL, "NULL array");
    TRY(ensure_device(h));
    if (mem_kind == BT_MEM_HOST) {  // _check_bin, score_collision's sigma_t check
        for (int64_t i = 0; i < n; ++i) {
            if (kind == 1 && !(values[i] > 0.0)) {
                char r[48];
                r[py_repr(values[i], r)] = 0;
                return set_err(BT_EINVAL, "sigma_t must be positive, got %s", r);
            }
            if (elements[i] < 0 || elements[i] >= h->ne)
                return set_err(BT_EINDEX, "element %d out of range [0, %lld)", elements[i],
                               (long long)h->ne);
            if (groups[i] < 0 || groups[i] >= h->ngroups)
                return set_err(BT_EINDEX, "group %d out of range [0, %d)", groups[i], h->ngroups);
        }
    }
    int32_t *de = nullptr, *dg = nullptr;
    double *dw = nullptr, *dx = nullptr;
    const int32_t* pe = elements;
    const int32_t* pg = groups;
    const double* pw = weights;
    const double* px = values;
    if (mem_kind == BT_MEM_HOST) {
        TRY(dalloc(&de, n));
        TRY(dalloc(&dg, n));
        TRY(dalloc(&dw, n));
        TRY(dalloc(&dx, n));
        CK(cudaMemcpyAsync(de, elements, sizeof(int32_t) * n, cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpyAsync(dg, groups, sizeof(int32_t) * n, cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpyAsync(dw, weights, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpyAsync(dx, values, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
        pe = de; pg = dg; pw = dw; px = dx;
    } else {
        CK(cudaMemsetAsync(h->dcounters + 15, 0, sizeof(unsigned long long), h->stream));
        score_check_kernel<<<grid_for(n, 256), 256, 0, h->stream>>>(pe, pg, px, n, h->ne,
                                                                    h->ngroups, kind,
                                                                    h->dcounters + 15);
        unsigned long long f = 0;
        CK(cudaMemcpyAsync(&f, h->dcounters + 15, sizeof f, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (f & 2ull) return set_err(BT_EINVAL, "sigma_t must be positive");
        if (f & 1ull) return set_err(BT_EINDEX, "element or group out of range");
    }
    score_kernel<<<grid_for(n, 256), 256, 0, h->stream>>>(pe, pg, pw, px, n, h->ngroups, kind,
                                                          h->tally);
    cudaError_t err = cudaGetLastError();
    if (err == cudaSuccess) err = cudaStreamSynchronize(h->stream);
    if (de) { cudaFree(de); cudaFree(dg); cudaFree(dw); cudaFree(dx); }
    if (err != cudaSuccess) return set_err(BT_ECUDA, "bt_score: %s", cudaGetErrorString(err));
    return BT_OK;
}

bt_status bt_write_tally(bt_tally* h, int32_t which, const double* in, int64_t n) {
    if (h && h->multi) {  // the unfinalized batch lives on shard 0 + the others: write it to
        Multi* m = h->multi;  // shard 0 and clear the rest; the moments are mirrored
        if (n != h->ne * h->ngroups) return set_err(BT_EINVAL, "n must be E*G");
        return fan_out(m, [&](int r) -> bt_status {
            bt_tally* t = m->shard[(size_t)r];
            if (which == BT_TALLY_BATCH && r > 0) {
                TRY(ensure_device(t));
                CK(cudaMemset(t->tally, 0, sizeof(double) * n));
                return BT_OK;
            }
            return bt_write_tally(t, which, in, n);
        });
    }
    if (!h || !in) return set_err(BT_EINVAL, "NULL argument");
    double* p = tally_ptr(h, which);
    if (!p) return set_err(BT_EINVAL, "unknown tally array %d", which);
    if (n != h->ne * h->ngroups) return set_err(BT_EINVAL, "n must be E*G");
    TRY(ensure_device(h));
    CK(cudaMemcpyAsync(p, in, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return BT_OK;
}

bt_status bt_set_batches_completed(bt_tally* h, int64_t n) {
    if (h && h->multi) {
        for (bt_tally* t : h->multi->shard) t->batches = n;
        return BT_OK;
    }
    if (!h || n < 0) return set_err(BT_EINVAL, "bad argument");
    h->batches = n;
    return BT_OK;
}

// ---- native mesh ingest (mesh.py:109-148, 302-331) and the paper-level ABI

bt_status bt_mesh_from_arrays(const double* vertices, int64_t num_vertices,
                              const int32_t* elements, int64_t num_elements, int32_t device,
                              bt_mesh** out) {
    if (!out) return set_err(BT_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_vertices < 0 || num_elements < 0) return set_err(BT_EINVAL, "negative size");
    if ((num_vertices && !vertices) || (num_elements && !elements))
        return set_err(BT_EINVAL, "NULL array");
    bt_mesh* m = new bt_mesh();
    m->nv = num_vertices;
    m->ne = num_elements;
    m->v.assign(vertices, vertices + 3 * num_vertices);
    m->e.assign(elements, elements + 4 * num_elements);
    const bt_status st = mesh_finish(m, device);
    if (st != BT_OK) {
        delete m;
        return st;
    }
    *out = m;
    return BT_OK;
}

bt_status bt_mesh_read(const char* path, int32_t device, bt_mesh** out) {
    if (!out || !path) return set_err(BT_EINVAL, "NULL argument");
    *out = nullptr;
    FILE* f = fopen(path, "rb");
    if (!f) return set_err(BT_EINVAL, "%s: cannot open", path);
    std::string data;
    fseek(f, 0, SEEK_END);
    const long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    data.resize(sz > 0 ? (size_t)sz : 0);
    const size_t got = sz > 0 ? fread(&data[0], 1, (size_t)sz, f) : 0;
    fclose(f);
    if ((long)got != sz) return set_err(BT_EINVAL, "%s: short read", path);
    bt_mesh* m = new bt_mesh();
    bt_status st = mesh_parse(path, data.data(), data.size(), m);
    if (st == BT_OK) st = mesh_finish(m, device);
    if (st != BT_OK) {
        delete m;
        return st;
    }
    *out = m;
    return BT_OK;
}

bt_status bt_mesh_info(const bt_mesh* m, int64_t* num_vertices, int64_t* num_elements) {
    if (!m) return set_err(BT_EINVAL, "NULL mesh");
    if (num_vertices) *num_vertices = m->nv;
    if (num_elements) *num_elements = m->ne;
    return BT_OK;
}

bt_status bt_mesh_arrays(const bt_mesh* m, double* vertices, int32_t* elements, int32_t* adj_elem,
                         int8_t* adj_face, double* volumes, double* centroids, double* bbox) {
    if (!m) return set_err(BT_EINVAL, "NULL mesh");
    auto cp = [](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) memcpy(dst, src, bytes);
    };
    cp(vertices, m->v.data(), sizeof(double) * m->v.size());
    cp(elements, m->e.data(), sizeof(int32_t) * m->e.size());
    cp(adj_elem, m->ae.data(), sizeof(int32_t) * m->ae.size());
    cp(adj_face, m->af.data(), m->af.size());
    cp(volumes, m->vol.data(), sizeof(double) * m->vol.size());
    cp(centroids, m->cen.data(), sizeof(double) * m->cen.size());
    cp(bbox, m->bbox, sizeof m->bbox);
    return BT_OK;
}

bt_status bt_mesh_destroy(bt_mesh* m) {
    delete m;
    return BT_OK;
}

bt_status bt_create_from_mesh(const bt_mesh* m, int64_t num_particles, int32_t num_groups,
                              int32_t device, bt_tally** out) {
    if (!m || !out) return set_err(BT_EINVAL, "NULL argument");
    if (m->ne == 0) return set_err(BT_EINVAL, "grid sizes must be positive");
    TRY(bt_create(m->v.data(), m->nv, m->e.data(), m->ae.data(), m->af.data(), m->ne, m->bbox,
                  m->cen.data(), num_particles, num_groups, device, out));
    (*out)->host_mesh = new bt_mesh(*m);
    return BT_OK;
}

bt_status bt_create_from_file(const char* mesh_filename, int64_t num_particles,
                              int32_t num_groups, int32_t device, bt_tally** out) {
    if (!out) return set_err(BT_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_particles <= 0) return set_err(BT_EINVAL, "num_particles must be positive");
    bt_mesh* m = nullptr;
    TRY(bt_mesh_read(mesh_filename, device, &m));
    const bt_status st = bt_create_from_mesh(m, num_particles, num_groups, device, out);
    bt_mesh_destroy(m);
    return st;
}

// the handle's mesh on the host: its own copy, or read back from the device
static bt_status handle_mesh(bt_tally* h, std::vector<double>& v, std::vector<int32_t>& e) {
    if (h->host_mesh) {
        v = h->host_mesh->v;
        e = h->host_mesh->e;
        return BT_OK;
    }
    bt_tally* s = h->multi ? h->multi->shard[0] : h;
    if (!s->vtx || !s->rec) return set_err(BT_EINVAL, "this handle has no mesh");
    TRY(ensure_device(s));
    std::vector<Vtx> hv((size_t)s->nv);
    std::vector<ElemRec> hr((size_t)s->ne);
    CK(cudaMemcpy(hv.data(), s->vtx, sizeof(Vtx) * hv.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), s->rec, sizeof(ElemRec) * hr.size(), cudaMemcpyDeviceToHost));
    v.resize((size_t)(3 * s->nv));
    e.resize((size_t)(4 * s->ne));
    for (int64_t i = 0; i < s->nv; ++i) {
        v[(size_t)(3 * i)] = hv[(size_t)i].x;
        v[(size_t)(3 * i + 1)] = hv[(size_t)i].y;
        v[(size_t)(3 * i + 2)] = hv[(size_t)i].z;
    }
    for (int64_t i = 0; i < s->ne; ++i)
        for (int k = 0; k < 4; ++k) e[(size_t)(4 * i + k)] = hr[(size_t)i].v[k];
    return BT_OK;
}

// flux (tally.py:123-152) of the handle's track-length moments, evaluated on
// the host in the reference's operation order (so the writers' text equals
// the reference writers' on the same moments)
static bt_status handle_flux(bt_tally* h, const double* volumes, std::vector<double>& mean,
                             std::vector<double>& rel) {
    const double* vol = volumes ? volumes : (h->host_mesh ? h->host_mesh->vol.data() : nullptr);
    if (!vol) return set_err(BT_EINVAL, "volumes are required for a handle made from arrays");
    int64_t n = 0;
    TRY(bt_batches_completed(h, &n));
    if (n == 0) return set_err(BT_ERUNTIME, "no batches completed; nothing to normalize");
    for (int64_t e = 0; e < h->ne; ++e)
        if (!(vol[e] > 0.0)) return set_err(BT_EINVAL, "volumes must be positive");
    const int64_t G = h->ngroups, nb = h->ne * G;
    std::vector<double> s((size_t)nb), sq((size_t)nb);
    TRY(bt_read_tally(h, BT_TALLY_SUM, s.data(), nb));
    TRY(bt_read_tally(h, BT_TALLY_SUM_SQ, sq.data(), nb));
    mean.assign((size_t)nb, 0.0);
    rel.assign((size_t)nb, 0.0);
    const double dn = (double)n;
    for (int64_t b = 0; b < nb; ++b) {
        const double bm = s[(size_t)b] / dn;
        mean[(size_t)b] = bm / vol[b / G];
        if (n >= 2) {
            double var = (sq[(size_t)b] - s[(size_t)b] * s[(size_t)b] / dn) / (dn - 1.0);
            if (var < 0.0) var = 0.0;  // np.clip(var, 0.0, None)
            const double se = std::sqrt(var / dn);
            if (bm > 0.0) rel[(size_t)b] = se / bm;
        }
    }
    return BT_OK;
}

bt_status bt_write_vtk(bt_tally* h, const char* filename, const double* volumes) {
    if (!h || !filename) return set_err(BT_EINVAL, "NULL argument");
    std::vector<double> mean, rel, v;
    std::vector<int32_t> e;
    TRY(handle_flux(h, volumes, mean, rel));
    TRY(handle_mesh(h, v, e));
    const int64_t nv = (int64_t)v.size() / 3, ne = (int64_t)e.size() / 4, G = h->ngroups;
    std::string s;
    s.reserve((size_t)(nv * 70 + ne * 60 + 2 * G * ne * 24 + 256));
    s += "# vtk DataFile Version 3.0\ntetrahedral mesh flux tally\nASCII\nDATASET UNSTRUCTURED_GRID\n";
    s += "POINTS " + std::to_string(nv) + " double\n";
    {
        char b[160];
        for (int64_t i = 0; i < nv; ++i) {
            int k = py_repr(v[(size_t)(3 * i)], b);
            b[k++] = ' ';
            k += py_repr(v[(size_t)(3 * i + 1)], b + k);
            b[k++] = ' ';
            k += py_repr(v[(size_t)(3 * i + 2)], b + k);
            b[k++] = '\n';
            s.append(b, (size_t)k);
        }
    }
    s += "CELLS " + std::to_string(ne) + " " + std::to_string(5 * ne) + "\n";
    {
        char b[80];
        for (int64_t i = 0; i < ne; ++i) {
            const int k = snprintf(b, sizeof b, "4 %d %d %d %d\n", e[(size_t)(4 * i)],
                                   e[(size_t)(4 * i + 1)], e[(size_t)(4 * i + 2)],
                                   e[(size_t)(4 * i + 3)]);
            s.append(b, (size_t)k);
        }
    }
    s += "CELL_TYPES " + std::to_string(ne) + "\n";
    for (int64_t i = 0; i < ne; ++i) s += "10\n";
    s += "CELL_DATA " + std::to_string(ne) + "\n";
    for (int64_t g = 0; g < G; ++g) {
        s += "SCALARS flux_g" + std::to_string(g) + " double 1\nLOOKUP_TABLE default\n";
        append_reprs(s, mean.data(), ne, G, g);
        s += "SCALARS rel_error_g" + std::to_string(g) + " double 1\nLOOKUP_TABLE default\n";
        append_reprs(s, rel.data(), ne, G, g);
    }
    return write_text(filename, s);
}

bt_status bt_write_flux_csv(bt_tally* h, const char* filename, const double* volumes) {
    if (!h || !filename) return set_err(BT_EINVAL, "NULL argument");
    std::vector<double> mean, rel;
    TRY(handle_flux(h, volumes, mean, rel));
    const int64_t ne = h->ne, G = h->ngroups;
    std::string s = "element,group,mean,rel_error\n";
    char b[128];
    for (int64_t e = 0; e < ne; ++e)
        for (int64_t g = 0; g < G; ++g) {
            int k = snprintf(b, sizeof b, "%lld,%lld,", (long long)e, (long long)g);
            k += py_repr(mean[(size_t)(e * G + g)], b + k);
            b[k++] = ',';
            k += py_repr(rel[(size_t)(e * G + g)], b + k);
            b[k++] = '\n';
            s.append(b, (size_t)k);
        }
    return write_text(filename, s);
}

bt_status bt_device_count(int32_t* n) {
    if (!n) return set_err(BT_EINVAL, "NULL argument");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *n = c;
    return BT_OK;
}

bt_status bt_format_double(double x, char* out, int32_t cap) {
    if (!out || cap < 32) return set_err(BT_EINVAL, "need a 32-byte buffer");
    const int k = py_repr(x, out);
    out[k] = 0;
    return BT_OK;
}

}  // extern "C"
