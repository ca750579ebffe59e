// b200tally.cu -- B200-native (sm_100a) tet-mesh walk with track-length
// tallies behind the C ABI declared in include/b200tally.h.
//
// Replaces the reference's numba hot path:
//   _sweep_fused + trace_and_score  search.py:169-275, 492-517 -> walk_kernel
//   initialize_locations            search.py:557-601          -> locate_grid_kernel
//                                                                 (or walk_kernel + tiebreak_kernel)
//   _tie_break_faces                search.py:520-551          -> tiebreak_kernel
//   _finalize                       tally.py:83-95              -> finalize_kernel
//   load_step                       particles.py:57-89          -> fused into walk_kernel's fetch
//
// Design: persistent CTAs, one particle per lane run to
// completion; idle lanes refill from a global work counter (warp-aggregated
// atomicAdd) so lanes stay busy despite the exponential crossings-per-move
// tail; the mesh is one 32-byte record per element (vertex ids + packed
// neighbour/face) plus 32-byte padded fp64 vertices, L2-resident up to ~3M
// tets; tallies are fp64 atomics into a private per-GPU grid, optionally
// aggregated per warp with __match_any_sync.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

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

// ---------------------------------------------------------------------------
// device data layout

struct __align__(32) ElemRec {
    int v[4];   // global vertex ids, reference local order (mesh.py:126-132)
    int nb[4];  // (neighbour << 2) | neighbour's local face, -1 on the boundary
};
static_assert(sizeof(ElemRec) == 32, "one 32-byte sector per element");

struct __align__(32) Vtx {
    double x, y, z, pad;
};
static_assert(sizeof(Vtx) == 32, "one 32-byte sector per vertex");

enum { C_EVENTS = 0, C_REACHED, C_BOUNDARY, C_RECOV, C_KILLED, C_SWEEPS, C_ERR, C_UNLOC, C_NCOUNTERS };
// dcounters layout (unsigned long long): [1..8] counters, [15] flags,
// [16 + c] queue of chunk c, [32 + c] work count of chunk c, c < MAX_CHUNKS
constexpr int MAX_CHUNKS = 16;
constexpr int NDCOUNTERS = 48;

// __match_any_sync aggregation of the tally atomics (BT_OPT_WARP_AGG)
enum { WAGG_ADAPTIVE = 0, WAGG_ALWAYS = 1, WAGG_NEVER = 2 };

struct WalkArgs {
    const ElemRec* __restrict__ rec;
    const Vtx* __restrict__ vtx;
    double* __restrict__ pos;            // (N,3) persistent
    const double* __restrict__ dest;     // (count,3) this move's destinations
    const int8_t* __restrict__ fly_in;   // (count) this move's flying flags
    const double* __restrict__ weight;   // (count) this move's weights (nullable if !score)
    const int32_t* __restrict__ group;   // (N) persistent groups
    int32_t* __restrict__ element;
    int8_t* __restrict__ alive;
    int8_t* __restrict__ entry;
    int8_t* __restrict__ stuck;
    int8_t* __restrict__ outcome;
    double* __restrict__ seg_total;
    double* __restrict__ tally;          // (E*G)
    uint64_t* __restrict__ digest;       // (N) nullable
    int64_t* __restrict__ dcount;        // (N) nullable
    const int32_t* __restrict__ order;   // (count) nullable: hand-out permutation
    unsigned long long* queue;
    unsigned long long* counters;        // C_NCOUNTERS
    int64_t count;
    int64_t max_sweeps;
    int32_t max_sweeps32;  // min(max_sweeps, INT32_MAX): the per-step guard's bound
    int32_t ngroups;
    int32_t score;
    int32_t wagg;    // tally atomics: WAGG_ADAPTIVE / WAGG_ALWAYS / WAGG_NEVER
};

__device__ __forceinline__ void load_tet(const WalkArgs& a, const ElemRec& r, Tet& T) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double2* p = reinterpret_cast<const double2*>(a.vtx + r.v[j]);
        const double2 xy = __ldg(p);
        const double2 zw = __ldg(p + 1);
        T.x[j] = xy.x;
        T.y[j] = xy.y;
        T.z[j] = zw.x;
    }
}

__device__ __forceinline__ ElemRec load_rec(const ElemRec* __restrict__ rec, int e) {
    const int4* p = reinterpret_cast<const int4*>(rec + e);
    const int4 a = __ldg(p);
    const int4 b = __ldg(p + 1);
    ElemRec r;
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    r.nb[0] = b.x; r.nb[1] = b.y; r.nb[2] = b.z; r.nb[3] = b.w;
    return r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// walk kernels: the fused sweep (search.py:169-275) run to completion per lane

constexpr int DEFAULT_VARIANT = 6;  // see run_walk's variant table

// Cold per-lane state (read at events and at the end of a walk) lives in
// shared memory, one slot per thread: fewer live registers in the hot loop.
constexpr int MAX_CTA_THREADS = 256;
__shared__ double s_lane_w[MAX_CTA_THREADS];
__shared__ double s_lane_seg[MAX_CTA_THREADS];
__shared__ int64_t s_lane_idx[MAX_CTA_THREADS];
__shared__ int s_lane_g[MAX_CTA_THREADS];
__shared__ double s_lane_d[3][MAX_CTA_THREADS];  // destination
__shared__ int8_t s_lane_outcome[MAX_CTA_THREADS];
__shared__ int8_t s_lane_alive[MAX_CTA_THREADS];

// one particle's walk state while it flies
struct Lane {
    ElemRec nr;   // prefetched record of the element entered next
    bool have_nr;
    bool busy;    // false: lane idle
    double px, py, pz;
    int e, entry, st, iters;
    __device__ __forceinline__ double& w() { return s_lane_w[threadIdx.x]; }
    __device__ __forceinline__ double& seg() { return s_lane_seg[threadIdx.x]; }
    __device__ __forceinline__ int64_t& idx() { return s_lane_idx[threadIdx.x]; }
    __device__ __forceinline__ int& g() { return s_lane_g[threadIdx.x]; }
    __device__ __forceinline__ int8_t& outcome() { return s_lane_outcome[threadIdx.x]; }
    __device__ __forceinline__ int8_t& alive() { return s_lane_alive[threadIdx.x]; }
    __device__ __forceinline__ double& dx() { return s_lane_d[0][threadIdx.x]; }
    __device__ __forceinline__ double& dy() { return s_lane_d[1][threadIdx.x]; }
    __device__ __forceinline__ double& dz() { return s_lane_d[2][threadIdx.x]; }
    __device__ __forceinline__ void set_idx(int64_t i) {
        idx() = i;
        busy = true;
    }
};

// this thread's digest slot in shared memory (digest mode only; keeps the
// sequence hash out of the hot loop's registers)
struct DigestSlot {
    uint64_t* d;
    int* c;
};

// Per-lane event count in a register; the rarer counters live in a
// CTA-shared array (fewer live registers in the hot loop), flushed once.
enum { SC_REACHED = 0, SC_BOUNDARY, SC_RECOV, SC_KILLED, SC_MAXIT, SC_ERR, SC_N };
struct Counters {
    unsigned events = 0;
    unsigned maxit = 0;      // longest walk (sweeps) finished by this lane
    unsigned* sh = nullptr;  // SC_N shared counters of the CTA
};

// Deferred track-length score of the previous step: its square root and
// atomic are issued after the next step's loads, off the critical path.
struct Pending {
    bool has = false;
    int64_t bin = 0;
    double val = 0.0;
    double seg = 0.0;
    bool seg_pending = false;
    int probe = 0;      // loop iterations to the next contention probe
    bool agg = false;   // warp-uniform: aggregate the pending scores
};

// One step of search.py:183-274 for a flying lane.  Returns true when the
// particle stops (reached, leaked, stuck-killed or sweep guard).  When DEFER
// the segment is left in P (scored by the next step or the loop); otherwise
// has_score/bin/val are set for an immediate score.
// DIG = false compiles the per-particle digest bookkeeping out of the loop.
template <bool DIG = true>
__device__ __forceinline__ bool walk_step(const WalkArgs& a, Lane& L, Counters& C, Pending& P,
                                          const DigestSlot& DS) {
    if (!L.have_nr) L.nr = load_rec(a.rec, L.e);  // not prefetched: first step after a hop
    const ElemRec r = L.nr;
    L.have_nr = false;
    Tet T;
    load_tet(a, r, T);
    // the previous step's score and seg_total update, while this step's
    // vertex loads are in flight (warp-aggregated mode scores at loop level)
    if (P.has) {  // not taken by an aggregated flush at loop level
        atomicAdd(a.tally + P.bin, P.val);
        P.has = false;
    }
    if (P.seg_pending) {
        L.seg() = __dadd_rn(L.seg(), P.seg);
        P.seg_pending = false;
    }
    double ox = L.px, oy = L.py, oz = L.pz;
    if (__builtin_expect(L.st == 1, 0)) {  // search.py:190-196
        const double sx = __dsub_rn(L.dx(), L.px), sy = __dsub_rn(L.dy(), L.py),
                     sz = __dsub_rn(L.dz(), L.pz);
        const double ln = __dsqrt_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(sx, sx), __dmul_rn(sy, sy)), __dmul_rn(sz, sz)));
        if (ln > 0.0) {
            ox = __dadd_rn(ox, __ddiv_rn(__dmul_rn(NUDGE, sx), ln));
            oy = __dadd_rn(oy, __ddiv_rn(__dmul_rn(NUDGE, sy), ln));
            oz = __dadd_rn(oz, __ddiv_rn(__dmul_rn(NUDGE, sz), ln));
        }
    }
    int face;
    double t;
    bool exact_used, need_t;
    int kind = exit_search_fast(T, ox, oy, oz, L.dx(), L.dy(), L.dz(), L.entry, &face, &t, &exact_used,
                                true, &need_t);
    // (neighbour << 2) | its face across the exit face, -1 on the boundary
    const int nbp = (face & 2) ? ((face & 1) ? r.nb[3] : r.nb[2]) : ((face & 1) ? r.nb[1] : r.nb[0]);
    if (kind == 1) {
        // issue the next element's record load now: it lands while the exact
        // t division and the commit below run
        if (nbp >= 0) {
            L.nr = load_rec(a.rec, nbp >> 2);
            L.have_nr = true;
        }
        if (need_t)
            t = exact_t(T, face, ox, oy, oz, rn_sub(L.dx(), ox), rn_sub(L.dy(), oy), rn_sub(L.dz(), oz));
    }
    bool done = false;
    bool event = true;
    if (kind == 2) {  // stuck ladder, search.py:199-235
        if (contains(T, L.dx(), L.dy(), L.dz(), STUCK_TOL)) {
            kind = 0;
            atomicAdd(C.sh + SC_RECOV, 1u);
        } else if (L.st == 0) {
            L.st = 1;
            atomicAdd(C.sh + SC_RECOV, 1u);
            event = false;
        } else if (L.st == 1) {
            int hop = -1;
#pragma unroll 1
            for (int f = 0; f < 4; ++f) {  // rare path: reload, no local arrays
                const int nbp = __ldg(&a.rec[L.e].nb[f]);
                if (hop < 0 && nbp >= 0) {
                    const int nb = nbp >> 2;
                    const ElemRec rn = load_rec(a.rec, nb);
                    Tet Tn;
                    load_tet(a, rn, Tn);
                    if (contains(Tn, ox, oy, oz, EPS_BARY)) hop = nb;
                }
            }
            event = false;
            if (hop >= 0) {
                L.e = hop;
                L.entry = -1;
                L.st = 2;
                atomicAdd(C.sh + SC_RECOV, 1u);
            } else {
                L.outcome() = OUT_STUCK_KILLED;
                L.alive() = 0;
                atomicAdd(C.sh + SC_KILLED, 1u);
                done = true;
            }
        } else {
            L.outcome() = OUT_STUCK_KILLED;
            L.alive() = 0;
            atomicAdd(C.sh + SC_KILLED, 1u);
            event = false;
            done = true;
        }
    }
    if (event) {  // search.py:236-274
        ++C.events;
        L.st = 0;
        if (DIG && a.digest) {
            *DS.d = (*DS.d ^ (uint64_t)((int64_t)L.e * 8 + face + 1)) * DIGEST_PRIME;
            ++*DS.c;
        }
        double qx, qy, qz;
        if (kind == 0) {
            qx = L.dx();
            qy = L.dy();
            qz = L.dz();
        } else {
            qx = __dadd_rn(ox, __dmul_rn(t, __dsub_rn(L.dx(), ox)));
            qy = __dadd_rn(oy, __dmul_rn(t, __dsub_rn(L.dy(), oy)));
            qz = __dadd_rn(oz, __dmul_rn(t, __dsub_rn(L.dz(), oz)));
        }
        const double ax = __dsub_rn(qx, L.px), ay = __dsub_rn(qy, L.py), az = __dsub_rn(qz, L.pz);
        const double seg = __dsqrt_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)), __dmul_rn(az, az)));
        P.has = a.score != 0;
        P.bin = (int64_t)L.e * a.ngroups + L.g();
        P.val = __dmul_rn(L.w(), seg);
        P.seg = seg;
        P.seg_pending = true;
        L.px = qx;
        L.py = qy;
        L.pz = qz;
        if (kind == 0) {
            L.entry = -1;
            L.outcome() = OUT_REACHED;
            atomicAdd(C.sh + SC_REACHED, 1u);
            done = true;
            // the particle stays in this element: a following flight (transport)
            // starts without the dependent record load
            L.nr = r;
            L.have_nr = true;
        } else {
            if (nbp < 0) {
                L.outcome() = OUT_LEAKED;
                L.alive() = 0;
                atomicAdd(C.sh + SC_BOUNDARY, 1u);
                done = true;
            } else {
                L.e = nbp >> 2;
                L.entry = nbp & 3;
            }
        }
    }
    ++L.iters;
    if (L.iters > a.max_sweeps32 && !done) {  // sweep guard, search.py:513-516
        atomicOr(C.sh + SC_ERR, 1u);
        done = true;
    }
    if (done && P.seg_pending) {  // the final seg_total is written now
        L.seg() = __dadd_rn(L.seg(), P.seg);
        P.seg_pending = false;
    }
    return done;
}

template <bool DIG = true>
__device__ __forceinline__ void finish(const WalkArgs& a, Lane& L, Counters& C,
                                       const DigestSlot& DS) {
    const int64_t i = L.idx();
    a.pos[3 * i] = L.px;
    a.pos[3 * i + 1] = L.py;
    a.pos[3 * i + 2] = L.pz;
    a.element[i] = L.e;
    a.entry[i] = (int8_t)L.entry;
    a.stuck[i] = (int8_t)L.st;
    a.outcome[i] = (int8_t)L.outcome();
    a.alive[i] = (int8_t)L.alive();
    a.seg_total[i] = L.seg();
    if (DIG && a.digest) {
        a.digest[i] = *DS.d;
        a.dcount[i] = *DS.c;
    }
    C.maxit = max(C.maxit, (unsigned)L.iters);
    L.busy = false;
}

template <bool DIG = true>
__device__ __forceinline__ void begin(Lane& L, const WalkArgs& a, const DigestSlot& DS) {
    L.have_nr = false;
    L.iters = 0;
    if (DIG && a.digest) {
        *DS.d = DIGEST_INIT;
        *DS.c = 0;
    }
    L.alive() = 1;          // overwritten by the fetch with alive | flying (load_step)
    L.outcome() = OUT_NONE;
}

// all lanes: one atomic per distinct bin of the warp's pending scores
__device__ __forceinline__ void score_aggregated(const WalkArgs& a, bool has_score, int64_t bin,
                                                 double val) {
    constexpr unsigned FULL = 0xffffffffu;
    {
        const int lane = threadIdx.x & 31;
        const unsigned m = __ballot_sync(FULL, has_score);
        if (has_score) {
            const unsigned peers = __match_any_sync(m, (unsigned long long)bin);
            const int leader = __ffs(peers) - 1;
            double sum = val;
            if (peers != (1u << lane)) {
                sum = 0.0;
                unsigned rest = peers;
                while (rest) {
                    const int src = __ffs(rest) - 1;
                    rest &= rest - 1;
                    sum = __dadd_rn(sum, __shfl_sync(peers, val, src));
                }
            }
            if (lane == leader) atomicAdd(a.tally + bin, sum);
        }
    }
}

// Loop level, all lanes converged.  Pending scores are normally left for the
// lane's next step to issue (after its loads, off the critical path).  They are
// aggregated here instead when the warp's lanes are scoring the same bins:
// always (WAGG_ALWAYS), or -- adaptive -- when a cheap probe (each lane's
// pending bin against the next lane's) finds a duplicate, which is what a point
// source with short flights produces (6x fewer contended atomics, measured in
// profiles/r01_options.jsonl).  Idle lanes flush their pending score.
__device__ __forceinline__ void flush_pending(const WalkArgs& a, Pending& P, bool idle) {
    constexpr unsigned FULL = 0xffffffffu;
    bool agg = a.wagg == WAGG_ALWAYS;
    if (a.wagg == WAGG_ADAPTIVE) {
        // probe every 4th iteration; the decision holds in between (warp-uniform)
        if (--P.probe <= 0) {
            const int lane = threadIdx.x & 31;
            const unsigned hm = __ballot_sync(FULL, P.has);
            const int nxt = __shfl_down_sync(FULL, (int)P.bin, 1);
            // low 32 bits: a false match only aggregates, which stays exact
            const bool dup = P.has && lane < 31 && ((hm >> (lane + 1)) & 1u) && nxt == (int)P.bin;
            P.agg = __any_sync(FULL, dup);
            P.probe = 4;
        }
        agg = P.agg;
    }
    if (agg) {
        score_aggregated(a, P.has, P.bin, P.val);
        P.has = false;
    } else if (idle && P.has) {
        atomicAdd(a.tally + P.bin, P.val);
        P.has = false;
    }
}

__device__ __forceinline__ void counters_init(unsigned* sh) {
    if (threadIdx.x < SC_N) sh[threadIdx.x] = 0;
    __syncthreads();
}

// all threads of the CTA: warp-reduce events, then one atomic per counter per CTA
__device__ __forceinline__ void flush_counters(const WalkArgs& a, Counters& C) {
    constexpr unsigned FULL = 0xffffffffu;
    const unsigned ev = __reduce_add_sync(FULL, C.events);
    if ((threadIdx.x & 31) == 0 && ev) atomicAdd(a.counters + C_EVENTS, (unsigned long long)ev);
    const unsigned mx = __reduce_max_sync(FULL, C.maxit);
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(C.sh + SC_MAXIT, mx);
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned* sh = C.sh;
        if (sh[SC_REACHED]) atomicAdd(a.counters + C_REACHED, (unsigned long long)sh[SC_REACHED]);
        if (sh[SC_BOUNDARY]) atomicAdd(a.counters + C_BOUNDARY, (unsigned long long)sh[SC_BOUNDARY]);
        if (sh[SC_RECOV]) atomicAdd(a.counters + C_RECOV, (unsigned long long)sh[SC_RECOV]);
        if (sh[SC_KILLED]) atomicAdd(a.counters + C_KILLED, (unsigned long long)sh[SC_KILLED]);
        if (sh[SC_MAXIT]) atomicMax(a.counters + C_SWEEPS, (unsigned long long)sh[SC_MAXIT]);
        if (sh[SC_ERR]) atomicOr(a.counters + C_ERR, 1ull);
    }
}

// v1: idle lanes refill straight from the particle arrays (one atomicAdd per
// warp per refill); the fetch's global loads sit on the step's critical path.
template <int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) walk_kernel(const WalkArgs a) {
    static_assert(THREADS <= MAX_CTA_THREADS, "one shared lane slot per thread");
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    __shared__ unsigned shc[SC_N];
    __shared__ uint64_t sdig[THREADS];
    __shared__ int scnt[THREADS];
    counters_init(shc);
    const DigestSlot DS{sdig + threadIdx.x, scnt + threadIdx.x};
    Lane L;
    L.busy = false;
    Counters C;
    C.sh = shc;
    Pending P;
    bool drained = false;
    while (true) {
        if (!drained) {
            const unsigned idle = __ballot_sync(FULL, !L.busy);
            if (idle) {
                const unsigned nidle = __popc(idle);
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(a.queue, (unsigned long long)nidle);
                base = __shfl_sync(FULL, base, 0);
                if (base + nidle >= (unsigned long long)a.count) drained = true;
                if (!L.busy) {
                    const unsigned long long q = base + __popc(idle & lanemask_lt());
                    if (q < (unsigned long long)a.count) {
                        const int64_t i = a.order ? (int64_t)a.order[q] : (int64_t)q;
                        if (a.digest && a.fly_in[i] == 0) {  // not moving: empty sequence
                            a.digest[i] = DIGEST_INIT;
                            a.dcount[i] = 0;
                        }
                        const bool unloc = a.fly_in[i] != 0 && a.element[i] < 0;
                        if (unloc) atomicAdd(a.counters + C_UNLOC, 1ull);
                        if (a.fly_in[i] != 0 && !unloc) {
                            L.set_idx(i);
                            L.e = a.element[i];
                            L.px = a.pos[3 * i];
                            L.py = a.pos[3 * i + 1];
                            L.pz = a.pos[3 * i + 2];
                            L.dx() = a.dest[3 * i];
                            L.dy() = a.dest[3 * i + 1];
                            L.dz() = a.dest[3 * i + 2];
                            L.entry = a.entry[i];
                            L.st = a.stuck[i];
                            L.seg() = a.seg_total[i];
                            L.w() = a.score ? a.weight[i] : 0.0;
                            L.g() = a.score ? a.group[i] : 0;
                            begin(L, a, DS);
                            L.alive() = (int8_t)(a.alive[i] | a.fly_in[i]);
                        }
                    }
                }
            }
        }
        if (!__any_sync(FULL, L.busy)) {
            flush_pending(a, P, true);
            if (drained) break;
            continue;
        }
        if (L.busy) {
            if (walk_step(a, L, C, P, DS)) finish(a, L, C, DS);
        }
        flush_pending(a, P, !L.busy);
    }
    flush_counters(a, C);
}

// ---------------------------------------------------------------------------
// v2: staged walk.  A stage kernel compacts the flying particles into SoA
// work arrays (coalesced); each warp then claims chunks of 32 work items and
// prefetches the NEXT chunk into shared memory with cp.async while its lanes
// keep walking, so refilling an idle lane is a shared-memory read instead of
// a dependent DRAM gather on the step's critical path.

struct WorkSoA {
    double *px, *py, *pz, *dx, *dy, *dz, *w, *seg;
    int *idx, *e, *g, *fl;  // fl = entry (low byte, signed) | stuck << 8
    int4 *r0, *r1;          // the starting element's record (vertex ids | adjacency)
};

// work items per stage chunk (one per lane at most).  Smaller chunks leave
// more of the SM's 256 KB to the L1 that caches the mesh gathers, but 8 and 16
// measured no faster than 32 on C2 (tools/build_variant.sh -DBT_STAGE_N=...)
#ifndef BT_STAGE_N
#define BT_STAGE_N 32
#endif
constexpr int STAGE_N = BT_STAGE_N;
static_assert(STAGE_N >= 1 && STAGE_N <= 32, "a stage chunk refills at most one warp");

struct __align__(16) WarpStage {
    double px[STAGE_N], py[STAGE_N], pz[STAGE_N], dx[STAGE_N], dy[STAGE_N], dz[STAGE_N],
        w[STAGE_N], seg[STAGE_N];
    int4 r0[STAGE_N], r1[STAGE_N];
    int idx[STAGE_N], e[STAGE_N], g[STAGE_N], fl[STAGE_N];
};


__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// claim the next chunk of 32 work items and start copying it into `st`;
// returns the number of valid items (warp-uniform)
__device__ __forceinline__ int claim_chunk(const WalkArgs& a, const WorkSoA& W, WarpStage& st,
                                           int64_t nwork) {
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(a.queue, (unsigned long long)STAGE_N);
    base = __shfl_sync(0xffffffffu, base, 0);
    const int64_t left = nwork - (int64_t)base;
    const int n = left <= 0 ? 0 : (left >= STAGE_N ? STAGE_N : (int)left);
    if (lane < n) {
        const int64_t k = (int64_t)base + lane;
        cp_async8(&st.px[lane], W.px + k);
        cp_async8(&st.py[lane], W.py + k);
        cp_async8(&st.pz[lane], W.pz + k);
        cp_async8(&st.dx[lane], W.dx + k);
        cp_async8(&st.dy[lane], W.dy + k);
        cp_async8(&st.dz[lane], W.dz + k);
        cp_async8(&st.w[lane], W.w + k);
        cp_async8(&st.seg[lane], W.seg + k);
        cp_async4(&st.idx[lane], W.idx + k);
        cp_async4(&st.e[lane], W.e + k);
        cp_async4(&st.g[lane], W.g + k);
        cp_async4(&st.fl[lane], W.fl + k);
        cp_async16(&st.r0[lane], W.r0 + k);
        cp_async16(&st.r1[lane], W.r1 + k);
    }
    cp_async_commit();
    return n;
}

template <int THREADS, int MINB, bool DIG>
__global__ void __launch_bounds__(THREADS, MINB)
    walk_staged_kernel(const WalkArgs a, const WorkSoA W, const int64_t* __restrict__ nwork_p) {
    static_assert(THREADS <= MAX_CTA_THREADS, "one shared lane slot per thread");
    constexpr unsigned FULL = 0xffffffffu;
    // the warps' double-buffered stages: dynamic shared memory (with the lane
    // slots the CTA exceeds the 48 KB static limit)
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    WarpStage(*stages)[2] = reinterpret_cast<WarpStage(*)[2]>(dyn_smem);
    __shared__ unsigned shc[SC_N];
    __shared__ uint64_t sdig[THREADS];
    __shared__ int scnt[THREADS];
    counters_init(shc);
    const DigestSlot DS{sdig + threadIdx.x, scnt + threadIdx.x};
    const int wid = threadIdx.x >> 5;
    const int64_t nwork = *nwork_p;
    Lane L;
    L.busy = false;
    Counters C;
    C.sh = shc;
    Pending P;
    int cur = 0;
    int head = 0;
    int ncur = claim_chunk(a, W, stages[wid][0], nwork);
    int nnext = ncur == STAGE_N ? claim_chunk(a, W, stages[wid][1], nwork) : 0;
    // only the first group must have landed; wait_group 1 would do, but the
    // second claim may be empty -- a full wait costs one DRAM latency once
    cp_async_wait_all();
    __syncwarp();
    while (true) {
        unsigned idle = __ballot_sync(FULL, !L.busy);
        while (idle) {
            if (head == ncur) {  // current stage used up: switch to the prefetched one
                if (nnext == 0) break;
                cp_async_wait_all();
                __syncwarp();
                cur ^= 1;
                head = 0;
                ncur = nnext;
                // the stage just emptied is free: prefetch the chunk after next
                nnext = (ncur == STAGE_N) ? claim_chunk(a, W, stages[wid][cur ^ 1], nwork) : 0;
            }
            const int take = min((int)__popc(idle), ncur - head);
            if (!L.busy) {
                const int rk = __popc(idle & lanemask_lt());
                if (rk < take) {
                    const WarpStage& s = stages[wid][cur];
                    const int j = head + rk;
                    L.set_idx(s.idx[j]);
                    L.px = s.px[j];
                    L.py = s.py[j];
                    L.pz = s.pz[j];
                    L.dx() = s.dx[j];
                    L.dy() = s.dy[j];
                    L.dz() = s.dz[j];
                    L.w() = s.w[j];
                    L.seg() = s.seg[j];
                    L.e = s.e[j];
                    L.g() = s.g[j];
                    const int fl = s.fl[j];
                    L.entry = (int)(signed char)(fl & 0xff);
                    L.st = (fl >> 8) & 0xff;
                    begin<DIG>(L, a, DS);
                    L.alive() = (int)(signed char)((fl >> 16) & 0xff);
                    // the first step's record came with the stage: no dependent load
                    const int4 q0 = s.r0[j], q1 = s.r1[j];
                    L.nr.v[0] = q0.x; L.nr.v[1] = q0.y; L.nr.v[2] = q0.z; L.nr.v[3] = q0.w;
                    L.nr.nb[0] = q1.x; L.nr.nb[1] = q1.y; L.nr.nb[2] = q1.z; L.nr.nb[3] = q1.w;
                    L.have_nr = true;
                }
            }
            head += take;
            idle = __ballot_sync(FULL, !L.busy);
        }
        if (!__any_sync(FULL, L.busy)) {  // no work left anywhere for this warp
            flush_pending(a, P, true);
            break;
        }
        if (L.busy) {
            if (walk_step<DIG>(a, L, C, P, DS)) finish<DIG>(a, L, C, DS);
        }
        flush_pending(a, P, !L.busy);
    }
    cp_async_wait_all();
    flush_counters(a, C);
}

// Compact this move's flying particles into the work arrays (order of
// indices within a warp preserved; warps in arbitrary order).  Non-flying
// particles get an empty digest.
// Particles [lo, lo + a.count) of this move; work items go to W (already
// offset by the caller).  A flying particle with element < 0 is not staged
// and counted (the move then reports it); wsum (nullable) accumulates the
// flying particles' weights (device-resident inputs).
__global__ void stage_kernel(const WalkArgs a, const WorkSoA W, int64_t* __restrict__ nwork,
                             int64_t lo, double* __restrict__ wsum) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    bool fly = false;
    int64_t i = 0;
    double wv = 0.0;
    if (t < a.count) {
        i = a.order ? (int64_t)a.order[t] : lo + t;
        fly = a.fly_in[i] != 0;
        if (a.digest && !fly) {
            a.digest[i] = DIGEST_INIT;
            a.dcount[i] = 0;
        }
        if (fly && wsum) wv = a.weight[i];
        if (fly && a.element[i] < 0) {
            atomicAdd(a.counters + C_UNLOC, 1ull);
            fly = false;
        }
    }
    if (wsum) {
        for (int o = 16; o > 0; o >>= 1) wv += __shfl_xor_sync(0xffffffffu, wv, o);
        if (lane == 0 && wv != 0.0) atomicAdd(wsum, wv);
    }
    const unsigned m = __ballot_sync(0xffffffffu, fly);
    if (!m) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd((unsigned long long*)nwork, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (!fly) return;
    const int64_t k = (int64_t)base + __popc(m & lanemask_lt());
    W.idx[k] = (int)i;
    W.px[k] = a.pos[3 * i];
    W.py[k] = a.pos[3 * i + 1];
    W.pz[k] = a.pos[3 * i + 2];
    W.dx[k] = a.dest[3 * i];
    W.dy[k] = a.dest[3 * i + 1];
    W.dz[k] = a.dest[3 * i + 2];
    W.w[k] = a.score ? a.weight[i] : 0.0;
    W.seg[k] = a.seg_total[i];
    W.e[k] = a.element[i];
    W.g[k] = a.score ? a.group[i] : 0;
    W.fl[k] = ((int)(unsigned char)a.entry[i]) | ((int)(unsigned char)a.stuck[i] << 8) |
              ((int)(unsigned char)(a.alive[i] | a.fly_in[i]) << 16);  // load_step: alive |= flying
    const int4* rp = reinterpret_cast<const int4*>(a.rec + a.element[i]);
    W.r0[k] = __ldg(rp);
    W.r1[k] = __ldg(rp + 1);
}

// ---------------------------------------------------------------------------
// Transport: the reference's event loop (transport.run,
// transport.py:445-549) alternates flight / walk / collide over all flying
// particles.  Particles never interact and every random draw is keyed by
// (seed, batch, particle, block) (rng.py:58-64), so each particle's history
// is the same whether it is advanced event by event or to completion: one
// lane runs a whole history (flight -> walk with track-length scoring ->
// collision estimator + scatter/absorb -> ...) in a persistent kernel.

constexpr uint64_t PH_M0 = 0xD2E7470EE14C6C93ull, PH_M1 = 0xCA5A826395121157ull;
constexpr uint64_t PH_W0 = 0x9E3779B97F4A7C15ull, PH_W1 = 0xBB67AE8584CAA73Bull;
constexpr uint64_t PH_KEY1 = 0xD1B54A32D192ED03ull;
constexpr double TWO_PI = 2.0 * 3.141592653589793;

// philox4x64-10 block (rng.py:38-49) -> four uniforms in (0, 1] (rng.py:52-64)
__device__ __forceinline__ void uniform_block(uint64_t seed, uint64_t batch, uint64_t particle,
                                              uint64_t block, double u[4]) {
    uint64_t c0 = block, c1 = particle, c2 = batch, c3 = 0, k0 = seed, k1 = PH_KEY1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t hi0 = __umul64hi(PH_M0, c0), lo0 = PH_M0 * c0;
        const uint64_t hi1 = __umul64hi(PH_M1, c2), lo1 = PH_M1 * c2;
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += PH_W0;
        k1 += PH_W1;
    }
    const double s = 1.0 / 9007199254740992.0;
    u[0] = __dmul_rn(__dadd_rn((double)(c0 >> 11), 1.0), s);
    u[1] = __dmul_rn(__dadd_rn((double)(c1 >> 11), 1.0), s);
    u[2] = __dmul_rn(__dadd_rn((double)(c2 >> 11), 1.0), s);
    u[3] = __dmul_rn(__dadd_rn((double)(c3 >> 11), 1.0), s);
}

__global__ void philox_kat_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                  double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uniform_block(keys[4 * i], keys[4 * i + 1], keys[4 * i + 2], keys[4 * i + 3], out + 4 * i);
}

// isotropic direction from two uniforms (transport.py:172-178, 255-261)
__device__ __forceinline__ void iso_dir(double ua, double ub, double& x, double& y, double& z) {
    const double mu = __dsub_rn(__dmul_rn(2.0, ua), 1.0);
    const double phi = __dmul_rn(TWO_PI, ub);
    const double t = __dsub_rn(1.0, __dmul_rn(mu, mu));
    const double s = __dsqrt_rn(t > 0.0 ? t : 0.0);
    double sp, cp;
    sincos(phi, &sp, &cp);
    x = __dmul_rn(s, cp);
    y = __dmul_rn(s, sp);
    z = mu;
}

struct XSDev {
    const double* sigma_t;      // (G)
    const double* scatter_prob; // (G)
    const double* group_cdf;    // (G,G)
    int32_t ng;
};

struct TransportArgs {
    WalkArgs w;                 // mesh, particle state, track tally (w.tally)
    XSDev xs;
    double* col_tally;          // collision estimator (E*G)
    double* dir;                // (N,3)
    uint32_t* rng_block;        // (N)
    int32_t* group_rw;          // (N) groups (written)
    double* weight_rw;          // (N)
    const double* src;          // (n,3) source positions (located)
    unsigned* round_max;        // per-round max walk steps (sweeps), MAX_ROUNDS_TRACKED
    unsigned long long* tcount; // [0] collisions [1] rounds overflow [2] lost
    double* wsum;               // [0] leaked [1] absorbed [2] stuck [3] track length
    unsigned long long* queue;
    uint64_t seed, batch;
    int64_t n;
    int64_t max_rounds;
};

constexpr int MAX_ROUNDS_TRACKED = 1 << 20;

// per-batch source sampling (transport.py:154-181), blocks 0 and 1
__global__ void transport_source_kernel(TransportArgs a, double box0, double box1, double box2,
                                        double box3, double box4, double box5, int fixed,
                                        double fdx, double fdy, double fdz,
                                        double* __restrict__ stage) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    double u[4];
    uniform_block(a.seed, a.batch, i, 0, u);
    stage[3 * i] = __dadd_rn(box0, __dmul_rn(__dsub_rn(box3, box0), u[0]));
    stage[3 * i + 1] = __dadd_rn(box1, __dmul_rn(__dsub_rn(box4, box1), u[1]));
    stage[3 * i + 2] = __dadd_rn(box2, __dmul_rn(__dsub_rn(box5, box2), u[2]));
    double dx = fdx, dy = fdy, dz = fdz;
    if (!fixed) {
        double v[4];
        uniform_block(a.seed, a.batch, i, 1, v);
        iso_dir(v[0], v[1], dx, dy, dz);
    }
    a.dir[3 * i] = dx;
    a.dir[3 * i + 1] = dy;
    a.dir[3 * i + 2] = dz;
    a.weight_rw[i] = 1.0;
    a.group_rw[i] = 0;
    a.rng_block[i] = 2;
}

// one history per lane, persistent; refill from a global counter
template <int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) transport_kernel(const TransportArgs t) {
    static_assert(THREADS <= MAX_CTA_THREADS, "one shared lane slot per thread");
    constexpr unsigned FULL = 0xffffffffu;
    const WalkArgs& a = t.w;
    const int lane = threadIdx.x & 31;
    __shared__ unsigned shc[SC_N];
    counters_init(shc);
    const DigestSlot DS{nullptr, nullptr};
    Lane L;
    L.busy = false;
    Counters C;
    C.sh = shc;
    Pending P;
    double ux = 0, uy = 0, uz = 0;  // direction
    uint32_t rb = 0;
    int rounds = 0;
    unsigned collisions = 0;
    double leaked = 0, absorbed = 0, stuck_w = 0;
    bool drained = false;
    bool need_flight = false;
    while (true) {
        if (!drained) {
            const unsigned idle = __ballot_sync(FULL, !L.busy);
            if (idle) {
                const unsigned nidle = __popc(idle);
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(t.queue, (unsigned long long)nidle);
                base = __shfl_sync(FULL, base, 0);
                if (base + nidle >= (unsigned long long)t.n) drained = true;
                if (!L.busy) {
                    const unsigned long long q = base + __popc(idle & lanemask_lt());
                    if (q < (unsigned long long)t.n && a.alive[q]) {
                        const int64_t i = (int64_t)q;
                        L.set_idx(i);
                        L.e = a.element[i];
                        L.px = a.pos[3 * i];
                        L.py = a.pos[3 * i + 1];
                        L.pz = a.pos[3 * i + 2];
                        L.seg() = 0.0;
                        L.w() = t.weight_rw[i];
                        L.g() = t.group_rw[i];
                        ux = t.dir[3 * i];
                        uy = t.dir[3 * i + 1];
                        uz = t.dir[3 * i + 2];
                        rb = t.rng_block[i];
                        L.entry = -1;
                        L.st = 0;
                        L.have_nr = false;  // a new history: load its element's record
                        rounds = 0;
                        need_flight = true;
                    }
                }
            }
        }
        if (!__any_sync(FULL, L.busy)) {
            flush_pending(a, P, true);
            if (drained) break;
            continue;
        }
        if (L.busy) {
            if (need_flight) {  // _flight (transport.py:213-226)
                double u[4];
                uniform_block(t.seed, t.batch, (uint64_t)L.idx(), rb, u);
                ++rb;
                const double lc = __ddiv_rn(-log(u[0]), t.xs.sigma_t[L.g()]);
                L.dx() = __dadd_rn(L.px, __dmul_rn(lc, ux));
                L.dy() = __dadd_rn(L.py, __dmul_rn(lc, uy));
                L.dz() = __dadd_rn(L.pz, __dmul_rn(lc, uz));
                L.iters = 0;
                L.outcome() = OUT_NONE;
                L.alive() = 1;
                ++rounds;
                need_flight = false;
            }
            if (walk_step<false>(a, L, C, P, DS)) {
                // flight over: its walk took L.iters sweeps in round `rounds`
                if (rounds <= MAX_ROUNDS_TRACKED) atomicMax(t.round_max + rounds - 1, (unsigned)L.iters);
                bool stop = true;
                if (L.outcome() == OUT_REACHED) {  // _collide (transport.py:229-275)
                    const int g = L.g();
                    const double st_g = t.xs.sigma_t[g];
                    atomicAdd(t.col_tally + (int64_t)L.e * t.xs.ng + g, __ddiv_rn(L.w(), st_g));
                    ++collisions;
                    double u[4];
                    uniform_block(t.seed, t.batch, (uint64_t)L.idx(), rb, u);
                    ++rb;
                    if (u[0] <= t.xs.scatter_prob[g]) {
                        int gp = 0;
                        for (int j = 0; j < t.xs.ng; ++j) {
                            gp = j;
                            if (u[1] <= t.xs.group_cdf[g * t.xs.ng + j]) break;
                        }
                        iso_dir(u[2], u[3], ux, uy, uz);
                        L.g() = gp;
                        stop = false;
                        need_flight = true;
                        if (rounds >= t.max_rounds) {  // _MAX_ROUNDS guard (transport.py:531-533)
                            atomicOr(C.sh + SC_ERR, 1u);
                            stop = true;
                        }
                    } else {
                        L.alive() = 0;
                        L.outcome() = 5;  // OUTCOME_ABSORBED
                        absorbed += L.w();
                    }
                } else if (L.outcome() == OUT_LEAKED) {
                    leaked += L.w();
                } else if (L.outcome() == OUT_STUCK_KILLED) {
                    stuck_w += L.w();
                }
                if (stop) {
                    const int64_t i = L.idx();
                    a.pos[3 * i] = L.px;
                    a.pos[3 * i + 1] = L.py;
                    a.pos[3 * i + 2] = L.pz;
                    a.element[i] = L.e;
                    a.entry[i] = (int8_t)L.entry;
                    a.stuck[i] = (int8_t)L.st;
                    a.outcome[i] = (int8_t)L.outcome();
                    a.alive[i] = (int8_t)L.alive();
                    a.seg_total[i] = L.seg();
                    t.dir[3 * i] = ux;
                    t.dir[3 * i + 1] = uy;
                    t.dir[3 * i + 2] = uz;
                    t.rng_block[i] = rb;
                    t.group_rw[i] = L.g();
                    L.busy = false;
                }
            }
        }
        flush_pending(a, P, !L.busy);
    }
    // reduce the per-lane totals (tally sums are order-free up to rounding)
    for (int o = 16; o > 0; o >>= 1) {
        leaked += __shfl_xor_sync(FULL, leaked, o);
        absorbed += __shfl_xor_sync(FULL, absorbed, o);
        stuck_w += __shfl_xor_sync(FULL, stuck_w, o);
    }
    collisions = __reduce_add_sync(FULL, collisions);
    if (lane == 0) {
        if (leaked != 0.0) atomicAdd(t.wsum + 0, leaked);
        if (absorbed != 0.0) atomicAdd(t.wsum + 1, absorbed);
        if (stuck_w != 0.0) atomicAdd(t.wsum + 2, stuck_w);
        if (collisions) atomicAdd(t.tcount + 0, (unsigned long long)collisions);
    }
    flush_counters(a, C);
}

__global__ void sum_rounds_kernel(const unsigned* __restrict__ round_max, int64_t n,
                                  unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        s += round_max[r];
    s = __reduce_add_sync(0xffffffffu, (unsigned)s);  // per-warp (< 2^32 per warp chunk)
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

__global__ void seg_sum_kernel(const double* __restrict__ seg, const int8_t* __restrict__ alive0,
                               int64_t n, double* __restrict__ out) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += seg[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(out, s);
}

__global__ void count_alive_kernel(const int8_t* __restrict__ alive, int64_t n,
                                   unsigned long long* __restrict__ out) {
    unsigned c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        c += alive[i] != 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// ---------------------------------------------------------------------------
// Listing-1 callback path (search.py:278-489): lockstep
// sweeps with a host callback between the proposal and the commit.

struct SweepBufs {
    int32_t* active;      // (cap) flying particle ids, ascending
    int32_t* has_ev;      // (cap) per active slot
    int32_t* offs;        // (cap + 1) exclusive scan of has_ev
    // per active slot
    int32_t* s_elem;
    int8_t* s_face;
    double* s_start;      // (cap,3)
    double* s_end;        // (cap,3)
    double* s_len;
    int32_t* s_next;
    int8_t* s_entry;
    int8_t* s_done;
    // compacted events (the callback view)
    int64_t* e_particle;
    int32_t* e_elem;
    int8_t* e_face;
    double* e_start;
    double* e_end;
    double* e_len;
    int32_t* e_next;      // writable by the callback
    int8_t* e_done;       // writable by the callback
    int32_t* e_next_prop;
    int8_t* e_entry;
    int8_t* e_done_prop;
};

__global__ void select_flying_kernel(const int8_t* __restrict__ fly, int64_t n,
                                     int32_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = fly[i] != 0;
}

__global__ void scatter_active_kernel(const int32_t* __restrict__ flag,
                                      const int32_t* __restrict__ offs, int64_t n,
                                      int32_t* __restrict__ active) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && flag[i]) active[offs[i]] = (int32_t)i;
}

// _sweep_events (search.py:278-372): proposal + immediate stuck-ladder effects
__global__ void sweep_propose_kernel(const WalkArgs a, int8_t* __restrict__ fly,
                                     SweepBufs B, int64_t m) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int64_t i = B.active[k];
    B.has_ev[k] = 0;
    if (fly[i] == 0) return;
    const int e = a.element[i];
    const double px = a.pos[3 * i], py = a.pos[3 * i + 1], pz = a.pos[3 * i + 2];
    const double dx = a.dest[3 * i], dy = a.dest[3 * i + 1], dz = a.dest[3 * i + 2];
    const int st = a.stuck[i];
    double ox = px, oy = py, oz = pz;
    if (st == 1) {
        const double sx = __dsub_rn(dx, px), sy = __dsub_rn(dy, py), sz = __dsub_rn(dz, pz);
        const double ln = __dsqrt_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(sx, sx), __dmul_rn(sy, sy)), __dmul_rn(sz, sz)));
        if (ln > 0.0) {
            ox = __dadd_rn(ox, __ddiv_rn(__dmul_rn(NUDGE, sx), ln));
            oy = __dadd_rn(oy, __ddiv_rn(__dmul_rn(NUDGE, sy), ln));
            oz = __dadd_rn(oz, __ddiv_rn(__dmul_rn(NUDGE, sz), ln));
        }
    }
    const ElemRec r = load_rec(a.rec, e);
    Tet T;
    load_tet(a, r, T);
    int face;
    double t;
    bool ex;
    int kind = exit_search_fast(T, ox, oy, oz, dx, dy, dz, a.entry[i], &face, &t, &ex);
    if (kind == 2) {
        if (contains(T, dx, dy, dz, STUCK_TOL)) {
            kind = 0;
            atomicAdd(a.counters + C_RECOV, 1ull);
        } else if (st == 0) {
            a.stuck[i] = 1;
            atomicAdd(a.counters + C_RECOV, 1ull);
            return;
        } else if (st == 1) {
            int hop = -1;
            for (int f = 0; f < 4 && hop < 0; ++f) {
                const int nbp = r.nb[f];
                if (nbp >= 0) {
                    const ElemRec rn = load_rec(a.rec, nbp >> 2);
                    Tet Tn;
                    load_tet(a, rn, Tn);
                    if (contains(Tn, ox, oy, oz, EPS_BARY)) hop = nbp >> 2;
                }
            }
            if (hop >= 0) {
                a.element[i] = hop;
                a.entry[i] = -1;
                a.stuck[i] = 2;
                atomicAdd(a.counters + C_RECOV, 1ull);
                return;
            }
            fly[i] = 0;
            a.alive[i] = 0;
            a.outcome[i] = OUT_STUCK_KILLED;
            atomicAdd(a.counters + C_KILLED, 1ull);
            return;
        } else {
            fly[i] = 0;
            a.alive[i] = 0;
            a.outcome[i] = OUT_STUCK_KILLED;
            atomicAdd(a.counters + C_KILLED, 1ull);
            return;
        }
    }
    a.stuck[i] = 0;
    B.has_ev[k] = 1;
    B.s_elem[k] = e;
    B.s_start[3 * k] = px;
    B.s_start[3 * k + 1] = py;
    B.s_start[3 * k + 2] = pz;
    double qx, qy, qz;
    if (kind == 0) {
        qx = dx;
        qy = dy;
        qz = dz;
        B.s_face[k] = -1;
        B.s_next[k] = -1;
        B.s_entry[k] = -1;
        B.s_done[k] = 1;
    } else {
        qx = __dadd_rn(ox, __dmul_rn(t, __dsub_rn(dx, ox)));
        qy = __dadd_rn(oy, __dmul_rn(t, __dsub_rn(dy, oy)));
        qz = __dadd_rn(oz, __dmul_rn(t, __dsub_rn(dz, oz)));
        const int nbp = face == 0 ? r.nb[0] : face == 1 ? r.nb[1] : face == 2 ? r.nb[2] : r.nb[3];
        B.s_face[k] = (int8_t)face;
        B.s_next[k] = nbp < 0 ? -1 : (nbp >> 2);
        B.s_entry[k] = nbp < 0 ? -1 : (int8_t)(nbp & 3);
        B.s_done[k] = nbp < 0 ? 1 : 0;
    }
    const double ax = __dsub_rn(qx, px), ay = __dsub_rn(qy, py), az = __dsub_rn(qz, pz);
    B.s_len[k] = __dsqrt_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)), __dmul_rn(az, az)));
    B.s_end[3 * k] = qx;
    B.s_end[3 * k + 1] = qy;
    B.s_end[3 * k + 2] = qz;
}

__global__ void sweep_compact_kernel(SweepBufs B, int64_t m) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m || !B.has_ev[k]) return;
    const int64_t j = B.offs[k];
    B.e_particle[j] = B.active[k];
    B.e_elem[j] = B.s_elem[k];
    B.e_face[j] = B.s_face[k];
    for (int c = 0; c < 3; ++c) {
        B.e_start[3 * j + c] = B.s_start[3 * k + c];
        B.e_end[3 * j + c] = B.s_end[3 * k + c];
    }
    B.e_len[j] = B.s_len[k];
    B.e_next[j] = B.s_next[k];
    B.e_next_prop[j] = B.s_next[k];
    B.e_entry[j] = B.s_entry[k];
    B.e_done[j] = B.s_done[k];
    B.e_done_prop[j] = B.s_done[k];
}

// _commit_events (search.py:375-419)
__global__ void sweep_commit_kernel(const WalkArgs a, int8_t* __restrict__ fly, SweepBufs B,
                                    int64_t nev) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nev) return;
    const int64_t i = B.e_particle[j];
    const int e = B.e_elem[j];
    const double seg = B.e_len[j];
    if (a.score) atomicAdd(a.tally + (int64_t)e * a.ngroups + a.group[i], __dmul_rn(a.weight[i], seg));
    a.seg_total[i] = __dadd_rn(a.seg_total[i], seg);
    a.pos[3 * i] = B.e_end[3 * j];
    a.pos[3 * i + 1] = B.e_end[3 * j + 1];
    a.pos[3 * i + 2] = B.e_end[3 * j + 2];
    if (a.digest) {
        a.digest[i] = (a.digest[i] ^ (uint64_t)((int64_t)e * 8 + B.e_face[j] + 1)) * DIGEST_PRIME;
        a.dcount[i] += 1;
    }
    if (B.e_done[j] != 0) {
        fly[i] = 0;
        if (B.e_face[j] == -1) {
            a.outcome[i] = OUT_REACHED;
            a.entry[i] = -1;
            atomicAdd(a.counters + C_REACHED, 1ull);
        } else if (B.e_next_prop[j] < 0) {
            a.alive[i] = 0;
            a.outcome[i] = OUT_LEAKED;
            atomicAdd(a.counters + C_BOUNDARY, 1ull);
        } else {
            a.outcome[i] = 4;  // OUTCOME_KILLED (by the callback)
        }
    } else {
        const int nxt = B.e_next[j];
        if (nxt >= 0) {
            a.element[i] = nxt;
            a.entry[i] = nxt == B.e_next_prop[j] ? B.e_entry[j] : (int8_t)-1;
        } else {
            a.entry[i] = -1;
        }
    }
}

// load_step (particles.py:57-89): alive |= flying, flying[count:] = 0
__global__ void load_step_kernel(const int8_t* __restrict__ fly_in, int64_t count, int64_t cap,
                                 int8_t* __restrict__ fly, int8_t* __restrict__ alive) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cap) return;
    if (i < count) {
        const int8_t f = fly_in[i];
        fly[i] = f;
        alive[i] = (int8_t)(alive[i] | f);
    } else {
        fly[i] = 0;
    }
}

__global__ void fill_digest_kernel(uint64_t* __restrict__ d, int64_t* __restrict__ c,
                                   int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        d[i] = DIGEST_INIT;
        c[i] = 0;
    }
}

// flux (tally.py:123-152) on the device: mean = (sum/n)/V, rel = sqrt(var/n)/mean
__global__ void flux_kernel(const double* __restrict__ sum, const double* __restrict__ sum_sq,
                            const double* __restrict__ vol, int64_t ne, int32_t ng, int64_t n,
                            double* __restrict__ mean, double* __restrict__ rel) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= ne * ng) return;
    const double s = sum[b], sq = sum_sq[b];
    const double dn = (double)n;
    const double bm = __ddiv_rn(s, dn);
    mean[b] = __ddiv_rn(bm, vol[b / ng]);
    double r = 0.0;
    if (n >= 2) {
        double var = __ddiv_rn(__dsub_rn(sq, __ddiv_rn(__dmul_rn(s, s), dn)), (double)(n - 1));
        if (var < 0.0) var = 0.0;
        const double se = __dsqrt_rn(__ddiv_rn(var, dn));
        if (bm > 0.0) r = __ddiv_rn(se, bm);
    }
    rel[b] = r;
}

// ---------------------------------------------------------------------------
// localization: uniform grid of element bounding boxes

// Barycentric pre-filter record of an element (64 bytes, fp32):
// lambda_k(p) = w_k . (p - c) + lc_k for k = 1..3, lambda_0 = 1 - l1 - l2 - l3,
// with w_k the rows of the inverse of [v1-v0 v2-v0 v3-v0] (fp64, then rounded)
// and c the rounded centroid.  K bounds the reference's own rounding of its
// Cramer quotients relative to sum|lambda| (1e-14 x the element's quality
// ratio A^3/|det|); +inf for poorly conditioned or degenerate elements, whose
// candidates always take the exact test.
struct __align__(16) ElemLam {
    float4 w1;  // w_1.xyz, lc_1
    float4 w2;
    float4 w3;
    float4 c;   // c.xyz, K
};
static_assert(sizeof(ElemLam) == 64, "two 32-byte sectors per element");

struct GridDev {
    double org[3];
    double cs[3];
    int dims[3];
    const int* cell_start;  // ncells + 1
    const int* cand;        // element ids, ascending within a cell
};

__device__ __forceinline__ int grid_axis(double p, double org, double cs, int dim) {
    double f = floor((p - org) / cs);
    int i = (f < 0.0) ? 0 : (f >= (double)dim ? dim - 1 : (int)f);
    return i;
}

__global__ void elem_cells_count_kernel(const ElemRec* __restrict__ rec,
                                        const Vtx* __restrict__ vtx, int64_t ne, GridDev G,
                                        int* __restrict__ counts, int4* __restrict__ ranges_lo,
                                        int4* __restrict__ ranges_hi) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const ElemRec r = rec[e];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int j = 0; j < 4; ++j) {
        const Vtx v = vtx[r.v[j]];
        const double c[3] = {v.x, v.y, v.z};
        for (int k = 0; k < 3; ++k) {
            lo[k] = fmin(lo[k], c[k]);
            hi[k] = fmax(hi[k], c[k]);
        }
    }
    double ext = fmax(fmax(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
    double delta = 1e-7 * ext + 1e-300;
    int a[3], b[3];
    for (int k = 0; k < 3; ++k) {
        a[k] = grid_axis(lo[k] - delta, G.org[k], G.cs[k], G.dims[k]);
        b[k] = grid_axis(hi[k] + delta, G.org[k], G.cs[k], G.dims[k]);
    }
    counts[e] = (b[0] - a[0] + 1) * (b[1] - a[1] + 1) * (b[2] - a[2] + 1);
    ranges_lo[e] = make_int4(a[0], a[1], a[2], 0);
    ranges_hi[e] = make_int4(b[0], b[1], b[2], 0);
}

__global__ void elem_lambda_kernel(const ElemRec* __restrict__ rec, const Vtx* __restrict__ vtx,
                                   int64_t ne, ElemLam* __restrict__ lam) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const ElemRec r = rec[e];
    double x[4], y[4], z[4];
    for (int j = 0; j < 4; ++j) {
        const Vtx v = vtx[r.v[j]];
        x[j] = v.x;
        y[j] = v.y;
        z[j] = v.z;
    }
    double a[3][3];  // a[k] = v_{k+1} - v0
    for (int k = 0; k < 3; ++k) {
        a[k][0] = x[k + 1] - x[0];
        a[k][1] = y[k + 1] - y[0];
        a[k][2] = z[k + 1] - z[0];
    }
    auto cross = [](const double* u, const double* v, double* o) {
        o[0] = u[1] * v[2] - u[2] * v[1];
        o[1] = u[2] * v[0] - u[0] * v[2];
        o[2] = u[0] * v[1] - u[1] * v[0];
    };
    double n[3][3];
    cross(a[1], a[2], n[0]);  // w_1 * det
    cross(a[2], a[0], n[1]);  // w_2 * det
    cross(a[0], a[1], n[2]);  // w_3 * det
    const double det = a[0][0] * n[0][0] + a[0][1] * n[0][1] + a[0][2] * n[0][2];
    double A = 0.0;
    for (int k = 0; k < 3; ++k) A = fmax(A, fabs(a[k][0]) + fabs(a[k][1]) + fabs(a[k][2]));
    const double q = A * A * A / fabs(det);
    const float cx = (float)((x[0] + x[1] + x[2] + x[3]) * 0.25);
    const float cy = (float)((y[0] + y[1] + y[2] + y[3]) * 0.25);
    const float cz = (float)((z[0] + z[1] + z[2] + z[3]) * 0.25);
    float4 w[3];
    for (int k = 0; k < 3; ++k) {
        const double wx = n[k][0] / det, wy = n[k][1] / det, wz = n[k][2] / det;
        const double lc = wx * ((double)cx - x[0]) + wy * ((double)cy - y[0]) +
                          wz * ((double)cz - z[0]);
        w[k] = make_float4((float)wx, (float)wy, (float)wz, (float)lc);
    }
    const float K = (q <= 1e6) ? __double2float_ru(1e-14 * q) : INFINITY;  // NaN q -> inf
    ElemLam L;
    L.w1 = w[0];
    L.w2 = w[1];
    L.w3 = w[2];
    L.c = make_float4(cx, cy, cz, K);
    lam[e] = L;
}

__global__ void elem_cells_emit_kernel(int64_t ne, GridDev G, const int* __restrict__ offs,
                                       const int4* __restrict__ ranges_lo,
                                       const int4* __restrict__ ranges_hi,
                                       unsigned long long* __restrict__ keys) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int4 a = ranges_lo[e], b = ranges_hi[e];
    int k = offs[e];
    for (int i = a.x; i <= b.x; ++i)
        for (int j = a.y; j <= b.y; ++j)
            for (int l = a.z; l <= b.z; ++l) {
                const unsigned long long cell =
                    ((unsigned long long)i * G.dims[1] + j) * G.dims[2] + l;
                keys[k++] = (cell << 32) | (unsigned long long)e;
            }
}

__global__ void cell_start_kernel(const unsigned long long* __restrict__ keys, int64_t m,
                                  int64_t ncells, int* __restrict__ start,
                                  int* __restrict__ cand) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < m) cand[c] = (int)(keys[c] & 0xffffffffull);
    if (c > ncells) return;
    // lower_bound of (c << 32)
    const unsigned long long target = (unsigned long long)c << 32;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    start[c] = (int)lo;
}

struct LocateArgs {
    const ElemRec* __restrict__ rec;
    const Vtx* __restrict__ vtx;
    const ElemLam* __restrict__ lam;
    GridDev G;
    const double* __restrict__ target;  // (count,3)
    double* __restrict__ pos;
    int32_t* __restrict__ element;
    int8_t* __restrict__ alive;
    int8_t* __restrict__ entry;
    int8_t* __restrict__ stuck;
    int8_t* __restrict__ outcome;
    double* __restrict__ seg_total;
    double bbox[6];
    double c0[3];
    int64_t count;
    int64_t lo;  // locate_grid_kernel: first particle of this launch
};

// elem_contains(p, EPS_BARY) (geometry.py:149-154) decided from the element's
// fp32 barycentric record: +1 certainly contained, -1 certainly not, 0 unsure
// (run the exact-equivalent test).  Error of lambda_k^f against the exact
// barycentric of the reference's fp64 vectors: the point's rounding to fp32
// (u T_k, T_k = sum|w_ki||p_i|), d = p - c and the FMA chain (<= 4 u S_k,
// S_k = sum|w_ki||d_i|), w's rounding (1.01 u S_k) and lc's (u|lc_k|); lambda_0
// adds three subtractions.  The reference's own quotients differ from the
// exact barycentrics by <= K sum|lambda| (K from the element's conditioning).
// Decisions need 1.25x that margin beyond -EPS_BARY.
__device__ __forceinline__ int lambda_prefilter(const ElemLam* __restrict__ L, float q0, float q1,
                                                float q2) {
    constexpr float u = 5.9604645e-8f;
    const float4 W1 = __ldg(&L->w1), W2 = __ldg(&L->w2), W3 = __ldg(&L->w3), C = __ldg(&L->c);
    const float d0 = q0 - C.x, d1 = q1 - C.y, d2 = q2 - C.z;
    const float ad0 = fabsf(d0), ad1 = fabsf(d1), ad2 = fabsf(d2);
    const float ap0 = fabsf(q0), ap1 = fabsf(q1), ap2 = fabsf(q2);
    float l[3], e[3];
    const float4 Ws[3] = {W1, W2, W3};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float4 W = Ws[k];
        l[k] = __fmaf_rn(W.x, d0, __fmaf_rn(W.y, d1, __fmaf_rn(W.z, d2, W.w)));
        const float S = __fmaf_rn(fabsf(W.x), ad0, __fmaf_rn(fabsf(W.y), ad1, fabsf(W.z) * ad2));
        const float T = __fmaf_rn(fabsf(W.x), ap0, __fmaf_rn(fabsf(W.y), ap1, fabsf(W.z) * ap2));
        e[k] = u * __fmaf_rn(1.02f, T, __fmaf_rn(5.1f, S, 4.1f * fabsf(W.w)));
    }
    const float l0 = ((1.0f - l[0]) - l[1]) - l[2];
    const float sl = fabsf(l[0]) + fabsf(l[1]) + fabsf(l[2]);
    const float ref = C.w * (1.0f + sl + fabsf(l0));  // K * sum|lambda|, inf when K is
    const float e0 = e[0] + e[1] + e[2] + 3.03f * u * (1.0f + sl);
    constexpr float tol = (float)EPS_BARY;
    bool pass = true, fail = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float lk = k == 0 ? l0 : l[k - 1];
        const float m = 1.25f * ((k == 0 ? e0 : e[k - 1]) + ref);
        pass &= lk + tol > m;
        fail |= lk + tol < -m;
    }
    return fail ? -1 : (pass ? 1 : 0);
}

// Warp-parallel grid search (the north star's localization kernel): a group
// of G lanes serves one particle (32/G particles per warp).  The group's
// lanes take G of the cell's candidates at a time -- ascending element ids --
// so the candidates' gathers of one particle are in flight together instead
// of one after another.  Each candidate is decided from its 64-byte fp32
// barycentric record (lambda_prefilter, no vertex gathers); only candidates
// within rounding distance of a face run the exact-equivalent containment
// filter on the fp64 vertices.  The lowest lane with a hit in
// the first chunk that has one is the lowest-id containing element
// (pkg/tests/oracles.py:36-57 semantics), for every G.
constexpr int LOCATE_THREADS = 256;
template <int G>
__global__ void __launch_bounds__(LOCATE_THREADS) locate_grid_kernel(const LocateArgs a) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr unsigned GMASK = G == 32 ? FULL : ((1u << G) - 1u);
    const int lane = threadIdx.x & 31;
    const int gl = lane % G, gid = lane / G;
    const int64_t i =
        a.lo + (blockIdx.x * (int64_t)LOCATE_THREADS + threadIdx.x) / G;  // this group's particle
    const bool valid = i < a.count;
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
    if (valid) {
        p0 = a.target[3 * i];
        p1 = a.target[3 * i + 1];
        p2 = a.target[3 * i + 2];
    }
    const bool inside = valid && p0 >= a.bbox[0] && p0 <= a.bbox[3] && p1 >= a.bbox[1] &&
                        p1 <= a.bbox[4] && p2 >= a.bbox[2] && p2 <= a.bbox[5];
    const float q0 = __double2float_rn(p0), q1 = __double2float_rn(p1), q2 = __double2float_rn(p2);
    int s0 = 0, s1 = 0;
    if (inside) {
        const int ci = grid_axis(p0, a.G.org[0], a.G.cs[0], a.G.dims[0]);
        const int cj = grid_axis(p1, a.G.org[1], a.G.cs[1], a.G.dims[1]);
        const int ck = grid_axis(p2, a.G.org[2], a.G.cs[2], a.G.dims[2]);
        const int64_t cell = ((int64_t)ci * a.G.dims[1] + cj) * a.G.dims[2] + ck;
        s0 = __ldg(a.G.cell_start + cell);
        s1 = __ldg(a.G.cell_start + cell + 1);
    }
    int found = -1;
    bool done = false;
    for (int k0 = s0;; k0 += G) {
        const bool act = !done && k0 < s1;  // group-uniform
        if (!__any_sync(FULL, act)) break;
        int c = -1;
        bool hit = false;
        const int k = k0 + gl;
        if (act && k < s1) {
            c = __ldg(a.G.cand + k);
            const int pre = lambda_prefilter(a.lam + c, q0, q1, q2);
            hit = pre > 0;
            if (pre == 0) {
                const ElemRec r = load_rec(a.rec, c);
                Tet T;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double2* vp = reinterpret_cast<const double2*>(a.vtx + r.v[j]);
                    const double2 xy = __ldg(vp);
                    const double2 zw = __ldg(vp + 1);
                    T.x[j] = xy.x;
                    T.y[j] = xy.y;
                    T.z[j] = zw.x;
                }
                hit = contains_fast(T, p0, p1, p2, EPS_BARY);
            }
        }
        const unsigned gm = (__ballot_sync(FULL, hit) >> (gid * G)) & GMASK;
        const int src = gm ? gid * G + __ffs(gm) - 1 : lane;
        const int fc = __shfl_sync(FULL, c, src);
        if (act && gm) {
            found = fc;
            done = true;
        }
    }
    if (!valid) return;
    if (gl < 3 && gl < G) {
        const double pv = gl == 0 ? p0 : gl == 1 ? p1 : p2;
        // outside the bbox the reference leaves centroid 0 (search.py:579-583)
        a.pos[3 * i + gl] = (found >= 0 || inside) ? pv : a.c0[gl];
    }
    if (G < 3) {  // narrow groups: the group's first lane writes the rest of pos
        if (gl == 0)
            for (int d = G; d < 3; ++d) {
                const double pv = d == 1 ? p1 : p2;
                a.pos[3 * i + d] = (found >= 0 || inside) ? pv : a.c0[d];
            }
    }
    if (gl == G - 1) {
        a.element[i] = found;
        a.alive[i] = found >= 0 ? 1 : 0;
        a.entry[i] = -1;
        a.stuck[i] = 0;
        a.outcome[i] = found >= 0 ? OUT_REACHED : (inside ? OUT_LEAKED : OUT_NONE);
        a.seg_total[i] = 0.0;
    }
}


// walk-mode localization, step 1: search.py:577-591
__global__ void init_walk_prep_kernel(LocateArgs a, int8_t* __restrict__ fly) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.count) return;
    const double p0 = a.target[3 * i], p1 = a.target[3 * i + 1], p2 = a.target[3 * i + 2];
    const bool inside = p0 >= a.bbox[0] && p0 <= a.bbox[3] && p1 >= a.bbox[1] &&
                        p1 <= a.bbox[4] && p2 >= a.bbox[2] && p2 <= a.bbox[5];
    a.pos[3 * i] = a.c0[0];
    a.pos[3 * i + 1] = a.c0[1];
    a.pos[3 * i + 2] = a.c0[2];
    a.element[i] = inside ? 0 : -1;
    a.alive[i] = inside ? 1 : 0;
    fly[i] = inside ? 1 : 0;
    a.entry[i] = -1;
    a.stuck[i] = 0;
    a.outcome[i] = OUT_NONE;
    a.seg_total[i] = 0.0;
}

// walk-mode localization, step 2: lost reset + _tie_break_faces (search.py:595-600)
__global__ void tiebreak_kernel(LocateArgs a) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.count) return;
    const int8_t oc = a.outcome[i];
    if (oc == OUT_LEAKED || oc == OUT_STUCK_KILLED) a.element[i] = -1;
    if (a.alive[i] == 0 || a.element[i] < 0) return;
    const double px = a.pos[3 * i], py = a.pos[3 * i + 1], pz = a.pos[3 * i + 2];
    int e = a.element[i];
    bool moved = true;
    while (moved) {
        moved = false;
        const ElemRec r = load_rec(a.rec, e);
        Tet T;
        for (int j = 0; j < 4; ++j) {
            const Vtx v = a.vtx[r.v[j]];
            T.x[j] = v.x;
            T.y[j] = v.y;
            T.z[j] = v.z;
        }
        double l[4];
        if (bary(T, px, py, pz, l) == 0.0) break;
        for (int f = 0; f < 4; ++f) {
            if (l[f] <= EPS_BARY) {
                const int nbp = r.nb[f];
                const int nb = nbp >> 2;
                if (nbp >= 0 && nb < e) {
                    const ElemRec rn = load_rec(a.rec, nb);
                    Tet Tn;
                    for (int j = 0; j < 4; ++j) {
                        const Vtx v = a.vtx[rn.v[j]];
                        Tn.x[j] = v.x;
                        Tn.y[j] = v.y;
                        Tn.z[j] = v.z;
                    }
                    if (contains(Tn, px, py, pz, EPS_BARY)) {
                        e = nb;
                        moved = true;
                        break;
                    }
                }
            }
        }
    }
    a.element[i] = e;
}

// ---------------------------------------------------------------------------
// move preparation: localization check (+ group range + source weight for
// device-resident inputs)

__global__ void prepare_kernel(const int8_t* __restrict__ fly, const int32_t* __restrict__ element,
                               const int32_t* __restrict__ groups, int32_t ngroups,
                               const double* __restrict__ weight, int64_t count,
                               unsigned long long* __restrict__ flags,
                               double* __restrict__ wsum) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool unloc = false, badg = false;
    double wv = 0.0;
    if (i < count) {
        const bool f = fly[i] != 0;
        unloc = f && element[i] < 0;
        if (groups) badg = groups[i] < 0 || groups[i] >= ngroups;
        if (wsum && f) wv = weight[i];
    }
    if (__any_sync(0xffffffffu, unloc) && (threadIdx.x & 31) == 0) atomicOr(flags, 1ull);
    if (__any_sync(0xffffffffu, badg) && (threadIdx.x & 31) == 0) atomicOr(flags, 2ull);
    if (wsum) {
        for (int o = 16; o > 0; o >>= 1) wv += __shfl_xor_sync(0xffffffffu, wv, o);
        if ((threadIdx.x & 31) == 0 && wv != 0.0) atomicAdd(wsum, wv);
    }
}

__global__ void finalize_kernel(double* __restrict__ acc, double* __restrict__ sum,
                                double* __restrict__ sum_sq, int64_t nbins, double w) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nbins) return;
    const double x = __ddiv_rn(acc[b], w);
    acc[b] = 0.0;
    sum[b] = __dadd_rn(sum[b], x);
    sum_sq[b] = __dadd_rn(sum_sq[b], __dmul_rn(x, x));
}

__global__ void iota_keys_kernel(const int32_t* __restrict__ element, int64_t count,
                                 unsigned* __restrict__ keys, int32_t* __restrict__ vals) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    keys[i] = (unsigned)(element[i] + 1);
    vals[i] = (int32_t)i;
}

// ---------------------------------------------------------------------------
// mesh ingest: face adjacency by two stable radix sorts (
// the reference builds it on the host with a lexsort, mesh.py:188-235)

__device__ __forceinline__ void face_triple(const int* __restrict__ el, int64_t row, int& a,
                                            int& b, int& c) {
    const int64_t e = row >> 2;
    const int f = (int)(row & 3);
    // face f = the three local vertices other than f (FACE_VERTICES, mesh.py:24-26)
    const int4 v = *reinterpret_cast<const int4*>(el + 4 * e);
    int x = f == 0 ? v.y : v.x;
    int y = f <= 1 ? v.z : v.y;
    int z = f == 3 ? v.z : v.w;
    // sort (x, y, z)
    int t;
    if (x > y) { t = x; x = y; y = t; }
    if (y > z) { t = y; y = z; z = t; }
    if (x > y) { t = x; x = y; y = t; }
    a = x; b = y; c = z;
}

__global__ void adj_keys_c_kernel(const int* __restrict__ el, int64_t nrows,
                                  unsigned* __restrict__ kc, int* __restrict__ rows) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    int a, b, c;
    face_triple(el, r, a, b, c);
    kc[r] = (unsigned)c;
    rows[r] = (int)r;
}

__global__ void adj_keys_ab_kernel(const int* __restrict__ el, int64_t nrows,
                                   const int* __restrict__ rows,
                                   unsigned long long* __restrict__ kab) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nrows) return;
    int a, b, c;
    face_triple(el, rows[k], a, b, c);
    kab[k] = ((unsigned long long)(unsigned)a << 32) | (unsigned)b;
}

// flags: 1 = face shared by 3+ elements (first sorted index in err[0]),
//        2 = element lists one face twice (element in err[1])
__global__ void adj_match_kernel(const int* __restrict__ el, int64_t nrows,
                                 const int* __restrict__ rows, int* __restrict__ adj_e,
                                 signed char* __restrict__ adj_f, unsigned* __restrict__ flags,
                                 long long* __restrict__ err) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k + 1 >= nrows) return;
    int a0, b0, c0, a1, b1, c1;
    face_triple(el, rows[k], a0, b0, c0);
    face_triple(el, rows[k + 1], a1, b1, c1);
    if (a0 != a1 || b0 != b1 || c0 != c1) return;
    if (k + 2 < nrows) {
        int a2, b2, c2;
        face_triple(el, rows[k + 2], a2, b2, c2);
        if (a2 == a0 && b2 == b0 && c2 == c0) {
            atomicOr(flags, 1u);
            atomicMin(err, (long long)k);
            return;
        }
    }
    if (k > 0) {
        int am, bm, cm;
        face_triple(el, rows[k - 1], am, bm, cm);
        if (am == a0 && bm == b0 && cm == c0) return;  // part of a 3-run, reported above
    }
    const int r0 = rows[k], r1 = rows[k + 1];
    const int e0 = r0 >> 2, f0 = r0 & 3, e1 = r1 >> 2, f1 = r1 & 3;
    if (e0 == e1) {
        atomicOr(flags, 2u);
        atomicMin(err + 1, (long long)e0);
        return;
    }
    adj_e[4 * (int64_t)e0 + f0] = e1;
    adj_f[4 * (int64_t)e0 + f0] = (signed char)f1;
    adj_e[4 * (int64_t)e1 + f1] = e0;
    adj_f[4 * (int64_t)e1 + f1] = (signed char)f0;
}

// duplicated element: all four faces shared with one and the same element
__global__ void adj_dup_kernel(const int* __restrict__ adj_e, int64_t ne,
                               unsigned* __restrict__ flags, long long* __restrict__ err) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int4 v = *reinterpret_cast<const int4*>(adj_e + 4 * e);
    if (v.x >= 0 && v.x == v.y && v.x == v.z && v.x == v.w) {
        atomicOr(flags, 4u);
        atomicMin(err + 2, (long long)e);
    }
}

// ---------------------------------------------------------------------------
// handle

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
    double* dwsum = nullptr;
    unsigned long long* hcounters = nullptr;  // pinned
    int move_chunks = 0;                      // host-input pipeline depth (0 = auto)
    int locate_lanes = 0;                     // grid search lanes per particle (0 = default)
    std::vector<double> host_sel;             // host scratch: weights of flying particles
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
    bool opt_staged = true;
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

static bt_status free_all(bt_tally* h) {
    void* ptrs[] = {h->rec, h->vtx, h->cell_start, h->cand, h->lam, h->pos, h->element, h->alive,
                    h->entry, h->stuck, h->outcome, h->seg_total, h->group, h->dest, h->fly,
                    h->weight, h->digest, h->dcount, h->order, h->sort_keys_in,
                    h->sort_keys_out, h->sort_vals_in, h->sort_tmp, h->tally, h->sum,
                    h->sum_sq, h->dcounters, h->dwsum, h->snap_pos, h->snap_element,
                    h->snap_flags, h->snap_seg, h->work_mem, h->init_stage,
                    h->col_tally, h->col_sum, h->col_sum_sq, h->tr_dir, h->tr_weight,
                    h->tr_rng, h->tr_round_max, h->tr_count, h->tr_wsum, h->tr_xs,
                    h->sb_mem, h->tr_fly, h->sb_flag, h->sb_tmp};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->hcounters) cudaFreeHost(h->hcounters);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->ev2) cudaEventDestroy(h->ev2);
    if (h->ev3) cudaEventDestroy(h->ev3);
    if (h->evc0) cudaEventDestroy(h->evc0);
    if (h->evc1) cudaEventDestroy(h->evc1);
    if (h->ev_loc) cudaEventDestroy(h->ev_loc);
    for (cudaEvent_t e : h->evchunk)
        if (e) cudaEventDestroy(e);
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
    // cells ~ E/6 over the bounding box, per-axis counts proportional to extent
    double ext[3];
    double vol = 1.0;
    for (int k = 0; k < 3; ++k) {
        ext[k] = h->bbox[3 + k] - h->bbox[k];
        if (!(ext[k] > 0.0)) ext[k] = 1e-300;
    }
    double maxext = std::max(ext[0], std::max(ext[1], ext[2]));
    for (int k = 0; k < 3; ++k) vol *= std::max(ext[k], 1e-6 * maxext);
    // cells per element (experiments: B200TALLY_GRID_DENSITY)
    double density = 0.5;  // measured best on C2 (profiles/r01_*): 3.9 ms / 1e7 points
    if (const char* env = getenv("B200TALLY_GRID_DENSITY")) density = std::max(1e-3, atof(env));
    double target = std::max(1.0, (double)h->ne * density);
    target = std::min(target, (double)(1 << 26));
    double cell = std::cbrt(vol / target);
    GridDev G{};
    int64_t ncells = 1;
    for (int k = 0; k < 3; ++k) {
        int d = (int)std::max(1.0, std::min(4096.0, std::round(ext[k] / cell)));
        if (ext[k] <= 1e-300) d = 1;
        G.dims[k] = d;
        G.org[k] = h->bbox[k];
        G.cs[k] = (ext[k] > 1e-300) ? ext[k] / d : 1.0;
        ncells *= d;
    }
    int* counts = nullptr;
    int* offs = nullptr;
    int4 *rlo = nullptr, *rhi = nullptr;
    TRY(dalloc(&counts, h->ne + 1));
    TRY(dalloc(&offs, h->ne + 1));
    TRY(dalloc(&rlo, h->ne));
    TRY(dalloc(&rhi, h->ne));
    CK(cudaMemsetAsync(counts + h->ne, 0, sizeof(int), h->stream));
    TRY(dalloc(&h->lam, h->ne));
    elem_cells_count_kernel<<<grid_for(h->ne, 256), 256, 0, h->stream>>>(h->rec, h->vtx, h->ne,
                                                                         G, counts, rlo, rhi);
    CK(cudaGetLastError());
    elem_lambda_kernel<<<grid_for(h->ne, 256), 256, 0, h->stream>>>(h->rec, h->vtx, h->ne, h->lam);
    CK(cudaGetLastError());
    size_t tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offs, (int)(h->ne + 1),
                                     h->stream));
    void* tmp = nullptr;
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offs, (int)(h->ne + 1), h->stream));
    int m = 0;
    CK(cudaMemcpyAsync(&m, offs + h->ne, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(tmp);
    unsigned long long *keys = nullptr, *keys_out = nullptr;
    TRY(dalloc(&keys, m));
    TRY(dalloc(&keys_out, m));
    elem_cells_emit_kernel<<<grid_for(h->ne, 256), 256, 0, h->stream>>>(h->ne, G, offs, rlo, rhi,
                                                                        keys);
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
    cudaFree(rlo);
    cudaFree(rhi);
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
    TRYF(dalloc(&h->dwsum, 1));
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

bt_status bt_destroy(bt_tally* h) {
    if (!h) return BT_OK;
    cudaSetDevice(h->dev);
    cudaStreamSynchronize(h->stream);
    cudaStreamSynchronize(h->cstream);
    free_all(h);
    delete h;
    return BT_OK;
}

bt_status bt_set_option(bt_tally* h, int32_t key, int64_t value) {
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
        case BT_OPT_STAGED: h->opt_staged = value != 0; break;
        case BT_OPT_MOVE_CHUNKS: h->move_chunks = (int)value; break;
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
    CK(cudaMalloc((void**)&p, n * (8 * sizeof(double) + 2 * sizeof(int4) + 4 * sizeof(int)) + 256));
    h->work_mem = p;
    WorkSoA& W = h->work;
    double* d = reinterpret_cast<double*>(p);
    W.px = d; W.py = d + n; W.pz = d + 2 * n; W.dx = d + 3 * n; W.dy = d + 4 * n;
    W.dz = d + 5 * n; W.w = d + 6 * n; W.seg = d + 7 * n;
    int4* r = reinterpret_cast<int4*>(d + 8 * n);
    W.r0 = r; W.r1 = r + n;
    int* q = reinterpret_cast<int*>(r + 2 * n);
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
    void (*staged)(const WalkArgs, const WorkSoA, const int64_t*);      // digests off
    void (*staged_dig)(const WalkArgs, const WorkSoA, const int64_t*);  // digests on
} kVariants[] = {
    // launch variant (CTA size, resident CTAs per SM = register budget);
    // BT_OPT_BLOCKS_PER_SM selects it, 0 = the tuned default
    {256, walk_kernel<256, 1>, walk_staged_kernel<256, 1, false>, walk_staged_kernel<256, 1, true>},  // 1: <=255 regs
    {256, walk_kernel<256, 2>, walk_staged_kernel<256, 2, false>, walk_staged_kernel<256, 2, true>},  // 2: <=128 regs
    {256, walk_kernel<256, 3>, walk_staged_kernel<256, 3, false>, walk_staged_kernel<256, 3, true>},  // 3: <=80 regs
    {128, walk_kernel<128, 3>, walk_staged_kernel<128, 3, false>, walk_staged_kernel<128, 3, true>},  // 4: <=168 regs
    {128, walk_kernel<128, 4>, walk_staged_kernel<128, 4, false>, walk_staged_kernel<128, 4, true>},  // 5: <=128 regs
    {192, walk_kernel<192, 2>, walk_staged_kernel<192, 2, false>, walk_staged_kernel<192, 2, true>},  // 6: <=168 regs
};

static WalkArgs walk_args(bt_tally* h, const double* dest, const int8_t* fly, const double* w,
                          bool score) {
    WalkArgs a;
    a.rec = h->rec;
    a.vtx = h->vtx;
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
    return a;
}

// zero the move's counters; the first walk launch records ev0
static bt_status walk_begin(bt_tally* h) {
    CK(cudaMemsetAsync(h->dcounters, 0, sizeof(unsigned long long) * NDCOUNTERS, h->stream));
    h->walk_first = true;
    return BT_OK;
}

// enqueue stage + walk of particles [lo, hi) as chunk `chunk` (staged path),
// or the whole range with the v1 kernel / element-sorted hand-out
static bt_status walk_enqueue(bt_tally* h, WalkArgs a, int64_t lo, int64_t hi, int chunk,
                              double* wsum, cudaStream_t st = nullptr) {
    if (!st) st = h->stream;
    const int64_t count = hi - lo;
    a.count = count;
    a.queue = h->dcounters + 16 + chunk;
    const bool staged = h->opt_staged;
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
    auto* staged_k = a.digest ? V.staged_dig : V.staged;
    const void* kptr = staged ? (const void*)staged_k : (const void*)V.plain;
    const size_t dyn = staged ? sizeof(WarpStage) * 2 * (V.threads / 32) : 0;
    if (staged) CK(cudaFuncSetAttribute(kptr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kptr, V.threads, dyn));
    bps = std::max(1, bps);
    const int64_t want = (count + V.threads - 1) / V.threads;
    const unsigned blocks =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)bps * h->num_sms));
    int64_t* nwork = reinterpret_cast<int64_t*>(h->dcounters + 32 + chunk);
    WorkSoA W = h->work;
    if (staged) {
        TRY(ensure_work(h));
        W = h->work;
        W.px += lo; W.py += lo; W.pz += lo; W.dx += lo; W.dy += lo; W.dz += lo;
        W.r0 += lo; W.r1 += lo;
        W.w += lo; W.seg += lo; W.idx += lo; W.e += lo; W.g += lo; W.fl += lo;
        stage_kernel<<<grid_for(count, 256), 256, 0, st>>>(a, W, nwork, lo, wsum);
        CK(cudaGetLastError());
        h->kernels += 1;
    }
    if (!staged && wsum) {  // the unstaged kernel has no stage pass to sum the weights in
        CK(cudaMemsetAsync(h->dcounters + 15, 0, sizeof(unsigned long long), st));
        prepare_kernel<<<grid_for(count, 256), 256, 0, st>>>(
            a.fly_in + lo, h->element + lo, nullptr, h->ngroups, a.weight + lo, count,
            h->dcounters + 15, wsum);
        CK(cudaGetLastError());
        h->kernels += 1;
    }
    if (h->walk_first) {
        CK(cudaEventRecord(h->ev0, st));
        h->walk_first = false;
    }
    if (staged)
        staged_k<<<blocks, V.threads, dyn, st>>>(a, W, nwork);
    else
        V.plain<<<blocks, V.threads, 0, st>>>(a);
    CK(cudaGetLastError());
    h->kernels += 1;
    return BT_OK;
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
static bt_status launch_locate(bt_tally* h, const LocateArgs& la, int64_t n) {
    const int g = h->locate_lanes > 0 ? h->locate_lanes : DEFAULT_LOCATE_LANES;
    const int64_t threads = n * g;
    const unsigned blocks = (unsigned)((threads + LOCATE_THREADS - 1) / LOCATE_THREADS);
    switch (g) {
        case 1: locate_grid_kernel<1><<<blocks, LOCATE_THREADS, 0, h->stream>>>(la); break;
        case 2: locate_grid_kernel<2><<<blocks, LOCATE_THREADS, 0, h->stream>>>(la); break;
        case 4: locate_grid_kernel<4><<<blocks, LOCATE_THREADS, 0, h->stream>>>(la); break;
        case 8: locate_grid_kernel<8><<<blocks, LOCATE_THREADS, 0, h->stream>>>(la); break;
        case 16: locate_grid_kernel<16><<<blocks, LOCATE_THREADS, 0, h->stream>>>(la); break;
        case 32: locate_grid_kernel<32><<<blocks, LOCATE_THREADS, 0, h->stream>>>(la); break;
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
    return a;
}

bt_status bt_initialize_particle_location(bt_tally* h, const double* positions, int64_t size,
                                          int32_t mem_kind, int32_t mode, bt_summary* summary) {
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
    if (host && mode == BT_LOCATE_GRID) {
        // Copy on the copy stream into a dedicated staging buffer, then
        // return as soon as the caller's buffer has been read: the
        // localization kernel runs on while the next call's copies proceed
        // (every later kernel or readout is ordered after it on `stream`).
        // Chunked: chunk c's localization starts as soon as its positions
        // have landed, while the next chunks are still being copied.
        if (!h->init_stage) TRY(dalloc(&h->init_stage, 3 * h->cap));
        CK(cudaStreamWaitEvent(h->cstream, h->ev_loc, 0));  // previous localization done
        const int nch = (int)std::min<int64_t>(count >= (4 << 20) ? 4 : 1, count);
        LocateArgs la = locate_args(h, h->init_stage, count);
        for (int c = 0; c < nch; ++c) {
            const int64_t lo = count * c / nch, hi = count * (c + 1) / nch;
            CK(cudaMemcpyAsync(h->init_stage + 3 * lo, positions + 3 * lo,
                               sizeof(double) * 3 * (hi - lo), cudaMemcpyHostToDevice,
                               h->cstream));
            CK(cudaEventRecord(h->evchunk[c], h->cstream));
            CK(cudaStreamWaitEvent(h->stream, h->evchunk[c], 0));
            la.lo = lo;
            la.count = hi;
            TRY(launch_locate(h, la, hi - lo));
        }
        CK(cudaEventRecord(h->evc0, h->cstream));
        CK(cudaEventRecord(h->ev_loc, h->stream));
        CK(cudaEventRecord(h->ev3, h->stream));
        CK(cudaEventSynchronize(h->evc0));
        h->call_pending = true;
        return BT_OK;
    }
    if (host) {
        CK(cudaMemcpyAsync(h->dest, positions, sizeof(double) * 3 * count,
                           cudaMemcpyHostToDevice, h->stream));
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

bt_status bt_move_to_next_location(bt_tally* h, const double* destinations, const int8_t* flying,
                                   const double* weights, const int32_t* groups, int64_t size,
                                   int32_t mem_kind, bt_summary* summary) {
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
        if (groups) {
            for (int64_t i = 0; i < count; ++i)
                if (groups[i] < 0 || groups[i] >= h->ngroups)
                    return set_err(BT_EINDEX, "group %d out of range [0, %d)", groups[i],
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
        // 1/8, 3/8, 1/2 for three) so the first walk starts after a short copy
        // and every later copy still finishes inside the previous chunk's walk.
        WalkArgs a = walk_args(h, h->dest, h->fly, h->weight, true);
        int nch = 1;
        if (h->opt_staged && !h->opt_sort) {
            nch = h->move_chunks > 0 ? h->move_chunks : (count >= (4 << 20) ? 3 : 1);
            nch = (int)std::min<int64_t>(std::min(nch, MAX_CHUNKS), count);
        }
        auto bound = [&](int c) -> int64_t {  // end of chunk c
            if (c + 1 >= nch) return count;
            const int sh = c == 0 ? nch : nch - 1 - c;
            return (int64_t)((double)count / (double)(1ll << sh));
        };
        TRY(walk_begin(h));
        // odd chunks go to a second stream, so chunk c+1's CTAs take the SMs
        // that chunk c's tail frees instead of waiting for its last walk
        CK(cudaEventRecord(h->ev_s1, h->stream));
        CK(cudaStreamWaitEvent(h->stream2, h->ev_s1, 0));
        for (int c = 0; c < nch; ++c) {
            const int64_t lo = c == 0 ? 0 : bound(c - 1), hi = bound(c);
            const int64_t n = hi - lo;
            if (n <= 0) continue;
            cudaStream_t st = (c & 1) ? h->stream2 : h->stream;
            CK(cudaMemcpyAsync(h->dest + 3 * lo, destinations + 3 * lo, sizeof(double) * 3 * n,
                               cudaMemcpyHostToDevice, h->cstream));
            CK(cudaMemcpyAsync(h->fly + lo, flying + lo, n, cudaMemcpyHostToDevice, h->cstream));
            CK(cudaMemcpyAsync(h->weight + lo, weights + lo, sizeof(double) * n,
                               cudaMemcpyHostToDevice, h->cstream));
            if (groups)
                CK(cudaMemcpyAsync(h->group + lo, groups + lo, sizeof(int32_t) * n,
                                   cudaMemcpyHostToDevice, h->cstream));
            CK(cudaEventRecord(h->evchunk[c], h->cstream));
            CK(cudaStreamWaitEvent(st, h->evchunk[c], 0));
            TRY(walk_enqueue(h, a, lo, hi, c, nullptr, st));
        }
        CK(cudaEventRecord(h->ev_s2, h->stream2));
        CK(cudaStreamWaitEvent(h->stream, h->ev_s2, 0));
        s = walk_end(h, a.max_sweeps, summary, ov);
        if (need_w) h->source_weight = job.out;
    } else {
        if (groups) {  // device groups: range check before any work
            CK(cudaMemcpyAsync(h->group, groups, sizeof(int32_t) * count,
                               cudaMemcpyDeviceToDevice, h->stream));
            CK(cudaMemsetAsync(h->dcounters + 15, 0, sizeof(unsigned long long), h->stream));
            prepare_kernel<<<grid_for(count, 256), 256, 0, h->stream>>>(
                flying, h->element, h->group, h->ngroups, weights, count, h->dcounters + 15,
                nullptr);
            CK(cudaGetLastError());
            h->kernels += 1;
            unsigned long long flags = 0;
            CK(cudaMemcpyAsync(&flags, h->dcounters + 15, sizeof flags, cudaMemcpyDeviceToHost,
                               h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (flags & 2ull) return set_err(BT_EINDEX, "group out of range [0, %d)", h->ngroups);
        }
        WalkArgs a = walk_args(h, destinations, flying, weights, true);
        if (need_w) CK(cudaMemsetAsync(h->dwsum, 0, sizeof(double), h->stream));
        TRY(walk_begin(h));
        TRY(walk_enqueue(h, a, 0, count, 0, need_w ? h->dwsum : nullptr));
        s = walk_end(h, a.max_sweeps, summary);
        if (need_w) {
            double dw = 0.0;
            CK(cudaMemcpy(&dw, h->dwsum, sizeof dw, cudaMemcpyDeviceToHost));
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
    if (!h || !ptr) return set_err(BT_EINVAL, "NULL argument");
    double* p = tally_ptr(h, which);
    if (!p) return set_err(BT_EINVAL, "unknown tally array %d", which);
    *ptr = p;
    return BT_OK;
}

bt_status bt_get_source_weight(bt_tally* h, double* w) {
    if (!h || !w) return set_err(BT_EINVAL, "NULL argument");
    *w = h->source_weight;
    return BT_OK;
}

bt_status bt_set_source_weight(bt_tally* h, double w) {
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    h->source_weight = w;
    return BT_OK;
}

bt_status bt_batches_completed(bt_tally* h, int64_t* n) {
    if (!h || !n) return set_err(BT_EINVAL, "NULL argument");
    *n = h->batches;
    return BT_OK;
}

bt_status bt_read_particles(bt_tally* h, int64_t count, double* position, int32_t* element,
                            int8_t* alive, int8_t* entry_face, int8_t* stuck, int8_t* outcome,
                            double* seg_total) {
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (count < 0 || count > h->cap) return set_err(BT_EINVAL, "count out of range");
    TRY(ensure_device(h));
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
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (!h->digest) return set_err(BT_EINVAL, "digests are off (BT_OPT_DIGEST)");
    if (count < 0 || count > h->cap) return set_err(BT_EINVAL, "count out of range");
    TRY(ensure_device(h));
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
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (position) *position = h->pos;
    if (element) *element = h->element;
    if (alive) *alive = h->alive;
    return BT_OK;
}

bt_status bt_save_state(bt_tally* h) {
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    TRY(ensure_device(h));
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
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (!h->have_snapshot) return set_err(BT_EINVAL, "no snapshot saved");
    TRY(ensure_device(h));
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
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (count < 0 || count > h->cap)
        return set_err(BT_EINVAL, "count %lld outside [0, %lld]", (long long)count,
                       (long long)h->cap);
    TRY(ensure_device(h));
    if (count == 0) return BT_OK;
    if (!destinations || !flying || !weights) return set_err(BT_EINVAL, "NULL array");
    if (!h->tr_fly) TRY(dalloc(&h->tr_fly, h->cap));
    const cudaMemcpyKind kind = mem_kind == BT_MEM_HOST ? cudaMemcpyHostToDevice
                                                        : cudaMemcpyDeviceToDevice;
    if (groups && mem_kind == BT_MEM_HOST)
        for (int64_t i = 0; i < count; ++i)
            if (groups[i] < 0 || groups[i] >= h->ngroups)
                return set_err(BT_EINDEX, "group %d out of range [0, %d)", groups[i], h->ngroups);
    CK(cudaMemcpyAsync(h->dest, destinations, sizeof(double) * 3 * count, kind, h->stream));
    CK(cudaMemcpyAsync(h->fly, flying, count, kind, h->stream));
    CK(cudaMemcpyAsync(h->weight, weights, sizeof(double) * count, kind, h->stream));
    if (groups)
        CK(cudaMemcpyAsync(h->group, groups, sizeof(int32_t) * count, kind, h->stream));
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
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    TRY(ensure_device(h));
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
    if (!h) return set_err(BT_EINVAL, "NULL handle");
    if (device) *device = h->dev;
    if (num_elements) *num_elements = h->ne;
    if (capacity) *capacity = h->cap;
    if (num_groups) *num_groups = h->ngroups;
    return BT_OK;
}

}  // extern "C"
