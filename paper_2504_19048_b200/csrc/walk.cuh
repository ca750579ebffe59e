// walk.cuh -- the walk kernels: lane state, walk_step, the staged persistent kernel, staging.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

// ---------------------------------------------------------------------------
// walk kernels: the fused sweep (search.py:169-275) run to completion per lane

constexpr int DEFAULT_VARIANT = 6;
// vertex slots per lane: the element's four, plus a scratch slot that the
// non-crossing lanes' zero-size copies land in (walk_step)
constexpr int NSLOT = 5;  // 192 x 2 CTAs/SM: see the launch variant table (b200tally.cu)

// Cold per-lane state (read only at the refill and at the end of a walk)
// lives in shared memory, one slot per thread.
#ifndef BT_MAX_CTA_THREADS
#define BT_MAX_CTA_THREADS 256
#endif
constexpr int MAX_CTA_THREADS = BT_MAX_CTA_THREADS;
__shared__ int64_t s_lane_idx[MAX_CTA_THREADS];
__shared__ int8_t s_lane_outcome[MAX_CTA_THREADS];
__shared__ int8_t s_lane_alive[MAX_CTA_THREADS];

// crossing record of one element, as held by a lane
struct XR {
    int nbp[4];
    unsigned nvs[4];
};
#ifndef BT_XR_V8
#define BT_XR_V8 1
#endif
__device__ __forceinline__ XR load_xr(const WalkArgs& a, int e) {
    XR r;
#if BT_XR_V8
    // one 256-bit load (LDG.E.ENL2.256): one L1TEX tag lookup per lane for the
    // whole 32-byte sector instead of two 128-bit loads (-0.7% on the C2 walk)
#ifndef BT_NO_L2_HINT
    asm("ld.global.nc.L2::cache_hint.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
        : "=r"(r.nbp[0]), "=r"(r.nbp[1]), "=r"(r.nbp[2]), "=r"(r.nbp[3]), "=r"(r.nvs[0]),
          "=r"(r.nvs[1]), "=r"(r.nvs[2]), "=r"(r.nvs[3])
        : "l"(a.xrec + e), "l"(mesh_policy()));
#else
    asm("ld.global.nc.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r.nbp[0]), "=r"(r.nbp[1]), "=r"(r.nbp[2]), "=r"(r.nbp[3]), "=r"(r.nvs[0]),
          "=r"(r.nvs[1]), "=r"(r.nvs[2]), "=r"(r.nvs[3])
        : "l"(a.xrec + e));
#endif
#else
    const int4* p = reinterpret_cast<const int4*>(a.xrec + e);
    const int4 u = ldg_mesh(p), v = ldg_mesh(p + 1);
    r.nbp[0] = u.x; r.nbp[1] = u.y; r.nbp[2] = u.z; r.nbp[3] = u.w;
    r.nvs[0] = v.x; r.nvs[1] = v.y; r.nvs[2] = v.z; r.nvs[3] = v.w;
#endif
    return r;
}
__device__ __forceinline__ void cpa8(unsigned dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
}
// cp.async of n (0 or 8) of 8 bytes: n = 0 zero-fills without reading global memory
__device__ __forceinline__ void cpa8n(unsigned dst, const void* src, unsigned n) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ double lds64(unsigned ad) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(ad));
    return v;
}

// one particle's walk state while it flies
struct Lane {
    XR nr;          // crossing record of element e (loaded one step ahead)
    unsigned pm;    // byte k = the shared-memory slot holding local vertex k
    unsigned vsb;   // this lane's vertex slots: x of slot 0 (shared address)
    unsigned vss;   // slot stride in bytes (coordinate stride = 4 * vss)
    bool busy;      // false: lane idle
    double px, py, pz;
    int e, entry, st, iters;
    // weight, group, seg_total and destination in registers: the peak
    // register use is in the exit filter, so they cost no occupancy, and
    // their shared-slot loads/stores cost 3% (seg_total) + 2.2% (the rest)
    double wr, segr, dxr, dyr, dzr;
    int gr;
    __device__ __forceinline__ double& w() { return wr; }
    __device__ __forceinline__ int& g() { return gr; }
    __device__ __forceinline__ double& seg() { return segr; }
    __device__ __forceinline__ double& dx() { return dxr; }
    __device__ __forceinline__ double& dy() { return dyr; }
    __device__ __forceinline__ double& dz() { return dzr; }
    __device__ __forceinline__ int64_t& idx() { return s_lane_idx[threadIdx.x]; }
    __device__ __forceinline__ int8_t& outcome() { return s_lane_outcome[threadIdx.x]; }
    __device__ __forceinline__ int8_t& alive() { return s_lane_alive[threadIdx.x]; }
    __device__ __forceinline__ void set_idx(int64_t i) {
        idx() = i;
        busy = true;
    }
};

// start copying element e's four vertices into the lane's slots (identity
// order) and load its crossing record; the next walk_step waits for them
__device__ __forceinline__ void vslots_fill(const WalkArgs& a, Lane& L, int e, const int4 v) {
    const int vid[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double* g = &a.vtx[vid[k]].x;
        const unsigned ad = L.vsb + k * L.vss;
        cpa8(ad, g);
        cpa8(ad + NSLOT * L.vss, g + 1);
        cpa8(ad + 2 * NSLOT * L.vss, g + 2);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    L.pm = 0x03020100u;
    L.nr = load_xr(a, e);
}
__device__ __forceinline__ int4 elem_vids(const WalkArgs& a, int e) {
    return ldg_mesh(reinterpret_cast<const int4*>(a.rec + e));
}
// shared-memory vertex slots of a kernel with THREADS threads
#define VSLOTS_DECL(THREADS)                                                   \
    __shared__ double s_vslots[3 * NSLOT * (THREADS)];                                \
    const unsigned vsb0 = (unsigned)__cvta_generic_to_shared(s_vslots + threadIdx.x); \
    constexpr unsigned VSS = 8u * (THREADS);
#define VSLOTS_INIT(L) \
    do {                  \
        (L).vsb = vsb0;   \
        (L).vss = VSS;    \
    } while (0)

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
    int probe = 0;      // loop iterations to the next contention probe
    bool agg = false;   // warp-uniform: aggregate the pending scores
    __device__ __forceinline__ void init(const WalkArgs& a) {
        agg = a.wagg == WAGG_ALWAYS;
        // one counter test per loop iteration in every mode: adaptive probes
        // on its first iteration, the fixed modes never (-1% against a mode
        // flag tested first)
        probe = a.wagg == WAGG_ADAPTIVE ? 0 : 0x7fffffff;
    }
};

// One step of search.py:183-274 for a flying lane.  Returns true when the
// particle stops (reached, leaked, stuck-killed or sweep guard).  The step's
// segment is left in P: scored at the start of the lane's next step -- the
// next step of the same particle or, after a refill, of the lane's next one --
// or by the loop-level flush.  DIG = false compiles the per-particle digest
// bookkeeping out of the loop.
template <bool DIG = true>
__device__ __forceinline__ bool walk_step(const WalkArgs& a, Lane& L, Counters& C, Pending& P,
                                          const DigestSlot& DS) {
    const XR r = L.nr;
    Tet T;
    // the previous step's score (warp-aggregated mode scores at loop level)
    // as a predicated reduction: no branch, the address is formed either way
    // (-0.35% on the C2 walk)
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p red.global.add.f64 [%0], %1;\n}"
                 ::"l"(a.tally + P.bin), "d"(P.val), "r"((unsigned)P.has) : "memory");
    P.has = false;
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
    // this element's vertices: three stayed in the lane's slots from the
    // previous element, the fourth was copied in (cp.async) when the previous
    // step chose its exit face -- one gather per crossing, issued a step
    // ahead.  Waited for only here, so the score atomic and the nudge check
    // above issue while the copy lands (in-order issue: -0.9%).
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const unsigned ad = L.vsb + ((L.pm >> (8 * k)) & 0xffu) * L.vss;
        T.x[k] = lds64(ad);
        T.y[k] = lds64(ad + NSLOT * L.vss);
        T.z[k] = lds64(ad + 2 * NSLOT * L.vss);
    }
    int face;
    double t;
    bool exact_used, need_t;
    int kind;
    if (DIG && a.exact_only) {  // validation: the reference's literal arithmetic only
        kind = exit_search(T, ox, oy, oz, L.dx(), L.dy(), L.dz(), L.entry, &face, &t);
        need_t = false;
    } else {
        kind = exit_search_fast(T, ox, oy, oz, L.dx(), L.dy(), L.dz(), L.entry, &face, &t,
                                &exact_used, true, &need_t);
    }
    // (neighbour << 2) | its face across the exit face, -1 on the boundary
    const int nbp = (face & 2) ? ((face & 1) ? r.nbp[3] : r.nbp[2]) : ((face & 1) ? r.nbp[1] : r.nbp[0]);
    {   // crossing: the neighbour's one new vertex replaces local vertex
        // `face` in its slot, and the slot map follows the neighbour's order.
        // Every lane issues the three copies (no branch: -1.4% on the C2
        // walk); the others copy zero bytes into their scratch slot
        const bool cross = kind == 1 && nbp >= 0;
        const int fc = face & 3;
        const unsigned nvs =
            (fc & 2) ? ((fc & 1) ? r.nvs[3] : r.nvs[2]) : ((fc & 1) ? r.nvs[1] : r.nvs[0]);
        const bool wide = a.xsel != nullptr;
        const int nv = wide ? (int)nvs : (int)(nvs & 0xffffffu);
        const unsigned s8 = wide ? (__ldg(a.xsel + L.e) >> (8 * fc)) & 0xffu : nvs >> 24;
        const unsigned t4 = (s8 | (s8 << 4)) & 0x0f0fu;
        const unsigned sel = (t4 | (t4 << 2)) & 0x3333u;
        const unsigned slot = cross ? (L.pm >> (8 * fc)) & 0xffu : 4u;
        const unsigned ad = L.vsb + slot * L.vss;
        const double* g = cross ? &a.vtx[nv].x : &a.vtx[0].x;
        const unsigned n = cross ? 8u : 0u;
        cpa8n(ad, g, n);
        cpa8n(ad + NSLOT * L.vss, g + 1, n);
        cpa8n(ad + 2 * NSLOT * L.vss, g + 2, n);
        asm volatile("cp.async.commit_group;\n" ::);
        L.pm = cross ? __byte_perm(L.pm, 0u, sel) : L.pm;
    }
    // the next step's crossing record: needed only after the next step's
    // exit filter, so its latency is hidden; the current element's again on
    // the paths where the particle stays (one definition, no register copies)
    L.nr = load_xr(a, (kind == 1 && nbp >= 0) ? (nbp >> 2) : L.e);
    {   // the exact t of the chosen face, evaluated by every lane without a
        // branch (-0.9% on the C2 walk): used where the fp32 filter decided a
        // crossing (t in (1e-12, 1], division in range); exact_t selects the
        // face's vertices, so any face value is safe for the other lanes
        const double tt = exact_t<true>(T, face, ox, oy, oz, rn_sub(L.dx(), ox),
                                        rn_sub(L.dy(), oy), rn_sub(L.dz(), oz));
        if (kind == 1 && need_t) t = tt;
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
                vslots_fill(a, L, hop, elem_vids(a, hop));
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
    {   // search.py:236-274, committed by every lane with selects (a step
        // without an event -- a stuck-ladder rung -- keeps its state); the
        // rare outcomes behind one branch (-0.85% on the C2 walk)
        C.events += event;
        L.st = event ? 0 : L.st;
        if (DIG && a.digest && event) {
            *DS.d = (*DS.d ^ (uint64_t)((int64_t)L.e * 8 + face + 1)) * DIGEST_PRIME;
            ++*DS.c;
        }
        const bool reach = kind == 0;
        const double qx = reach ? L.dx() : __dadd_rn(ox, __dmul_rn(t, __dsub_rn(L.dx(), ox)));
        const double qy = reach ? L.dy() : __dadd_rn(oy, __dmul_rn(t, __dsub_rn(L.dy(), oy)));
        const double qz = reach ? L.dz() : __dadd_rn(oz, __dmul_rn(t, __dsub_rn(L.dz(), oz)));
        const double ax = __dsub_rn(qx, L.px), ay = __dsub_rn(qy, L.py), az = __dsub_rn(qz, L.pz);
        const double seg = __dsqrt_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)), __dmul_rn(az, az)));
        P.has = event && a.score != 0;
        P.bin = (int64_t)L.e * a.ngroups + L.g();
        P.val = __dmul_rn(L.w(), seg);
        L.seg() = event ? __dadd_rn(L.seg(), seg) : L.seg();
        L.px = event ? qx : L.px;
        L.py = event ? qy : L.py;
        L.pz = event ? qz : L.pz;
        const bool ereach = event && reach, leak = event && !reach && nbp < 0;
        if (ereach || leak) {
            L.outcome() = ereach ? OUT_REACHED : OUT_LEAKED;
            if (leak) L.alive() = 0;
            atomicAdd(C.sh + (ereach ? SC_REACHED : SC_BOUNDARY), 1u);
            done = true;
        }
        const bool cross = event && !reach && nbp >= 0;
        L.e = cross ? nbp >> 2 : L.e;
        L.entry = cross ? (nbp & 3) : (ereach ? -1 : L.entry);
    }
    ++L.iters;
    // sweep guard (search.py:513-516): the reference raises once its sweep
    // count exceeds the limit, even when the last particle finished in that
    // very sweep -- so a lane finishing on step limit + 1 raises too.  The
    // walk just ends here (no branch per step); the error is flagged where a
    // walk ends (finish(), the transport's flight end: sweep_guard_hit)
    return done || L.iters > a.max_sweeps32;
}

// a walk ended: flag the sweep guard if it was the guard that ended it
__device__ __forceinline__ void sweep_guard_hit(const WalkArgs& a, const Lane& L, Counters& C) {
    if (L.iters > a.max_sweeps32) atomicOr(C.sh + SC_ERR, 1u);
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
    sweep_guard_hit(a, L, C);
    L.busy = false;
}

template <bool DIG = true>
__device__ __forceinline__ void begin(Lane& L, const WalkArgs& a, const DigestSlot& DS) {
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
#ifndef BT_AGG_HOLD
#define BT_AGG_HOLD 128
#endif
constexpr int AGG_HOLD = BT_AGG_HOLD;  // iterations aggregation stays on once a probe finds contention
__device__ __forceinline__ void flush_pending(const WalkArgs& a, Pending& P, bool idle) {
    constexpr unsigned FULL = 0xffffffffu;
    // mode flags resolved once per kernel (Pending::init); P.agg is the
    // current decision in every mode
    if (--P.probe <= 0) {  // probe every 4th iteration (warp-uniform; adaptive mode only)
        const int lane = threadIdx.x & 31;
        const unsigned hm = __ballot_sync(FULL, P.has);
        const int nxt = __shfl_down_sync(FULL, (int)P.bin, 1);
        // low 32 bits: a false match only aggregates, which stays exact
        const bool dup = P.has && lane < 31 && ((hm >> (lane + 1)) & 1u) && nxt == (int)P.bin;
        P.agg = __any_sync(FULL, dup);
        P.probe = P.agg ? AGG_HOLD : 4;
    }
    const bool agg = P.agg;
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
    if (!gate_open(a, false)) return;  // v1 launches never set gate_pick
    const int lane = threadIdx.x & 31;
    __shared__ unsigned shc[SC_N];
    __shared__ uint64_t sdig[THREADS];
    __shared__ int scnt[THREADS];
    VSLOTS_DECL(THREADS)
    counters_init(shc);
    const DigestSlot DS{sdig + threadIdx.x, scnt + threadIdx.x};
    Lane L;
    L.busy = false;
    VSLOTS_INIT(L);
    Counters C;
    C.sh = shc;
    Pending P;
    P.init(a);
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
                            vslots_fill(a, L, L.e, elem_vids(a, L.e));
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
    int4* r0;               // the starting element's vertex ids
};

// work items per stage chunk (one per lane at most).  Smaller chunks leave
// more of the SM's 256 KB to the L1 that caches the mesh gathers, but 8 and 16
// measured no faster than 32 on C2 (tools/build_variant.sh -DBT_STAGE_N=...)
#ifndef BT_STAGE_N
#define BT_STAGE_N 32
#endif
constexpr int STAGE_N = BT_STAGE_N;
#ifndef BT_REFILL_MIN
#define BT_REFILL_MIN 2
#endif
constexpr int REFILL_MIN = BT_REFILL_MIN;  // idle lanes that trigger a refill (staged walk)
static_assert(STAGE_N >= 1 && STAGE_N <= 32, "a stage chunk refills at most one warp");

struct __align__(16) WarpStage {
    double px[STAGE_N], py[STAGE_N], pz[STAGE_N], dx[STAGE_N], dy[STAGE_N], dz[STAGE_N],
        w[STAGE_N], seg[STAGE_N];
    int4 r0[STAGE_N];
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
    }
    cp_async_commit();
    return n;
}

// Direct refill (no stage kernel, no work list): a warp claims 32 consecutive
// slots of the move and reads its particles straight from the particle
// arrays into a stage (plain loads: one latency per 32 particles; measured
// faster than splitting them into cp.async groups), including the starting
// element's record.  Flags: bit 24 = walkable (flying and localized), bit 25
// = flying.
// a streamed move's warp gives up on inputs that have not landed after 5 s
constexpr unsigned long long STREAM_STALL_NS = 5000000000ull;
struct DirectArgs {
    int64_t lo, hi;  // particles [lo, hi) of this launch (slots through a.order if set)
};

__device__ __forceinline__ int claim_direct(const WalkArgs& a, const DirectArgs& d, WarpStage& st) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(a.queue, (unsigned long long)STAGE_N);
    base = __shfl_sync(FULL, base, 0);
    const int64_t left = (d.hi - d.lo) - (int64_t)base;
    const int n = left <= 0 ? 0 : (left >= STAGE_N ? STAGE_N : (int)left);
    if (a.ready && n > 0) {  // streamed host-input move: wait for this chunk's inputs
        int stalled = 0;
        if (lane == 0) {
            const unsigned long long need = (unsigned long long)(d.lo + (int64_t)base + n);
            unsigned long long r, t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            while (true) {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(r) : "l"(a.ready) : "memory");
                if (r >= need) break;
                __nanosleep(256);
                // inputs that never arrive (a tool that runs this launch alone,
                // say) end the walk with an error instead of a hung GPU
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > STREAM_STALL_NS) {
                    atomicOr(a.counters + C_ERR, 2ull);
                    stalled = 1;
                    break;
                }
            }
        }
        if (__shfl_sync(FULL, stalled, 0)) return 0;
    }
    if (lane < n) {
        const int64_t t = (int64_t)base + lane;
        const int64_t i = a.order ? (int64_t)a.order[t] : d.lo + t;
        const int fly = a.fly_in[i] != 0;
        const int el = a.element[i];
        const bool walk = fly && el >= 0;
        st.idx[lane] = (int)i;
        st.px[lane] = a.pos[3 * i];
        st.py[lane] = a.pos[3 * i + 1];
        st.pz[lane] = a.pos[3 * i + 2];
        st.dx[lane] = a.dest[3 * i];
        st.dy[lane] = a.dest[3 * i + 1];
        st.dz[lane] = a.dest[3 * i + 2];
        const double w = a.score ? a.weight[i] : 0.0;
        st.w[lane] = w;
        st.seg[lane] = a.seg_total[i];
        st.e[lane] = el;
        st.g[lane] = a.score ? a.group[i] : 0;
        st.fl[lane] = ((int)(unsigned char)a.entry[i]) | ((int)(unsigned char)a.stuck[i] << 8) |
                      ((int)(unsigned char)(a.alive[i] | a.fly_in[i]) << 16) |  // load_step
                      (walk ? 1 << 24 : 0) | (fly ? 1 << 25 : 0);
        if (walk) {
            const int4* rp = reinterpret_cast<const int4*>(a.rec + el);
            st.r0[lane] = ldg_mesh(rp);
        }
    }
    __syncwarp();
    return n;
}

// DIRECT: stages filled by claim_direct from the particle arrays; otherwise
// from the stage kernel's work list with cp.async (claim_chunk).
template <int THREADS, int MINB, bool DIG, bool DIRECT>
__global__ void __launch_bounds__(THREADS, MINB)
    walk_staged_kernel(const WalkArgs a, const WorkSoA W, const int64_t* __restrict__ nwork_p,
                       const DirectArgs D) {
    static_assert(THREADS <= MAX_CTA_THREADS, "one shared lane slot per thread");
    constexpr unsigned FULL = 0xffffffffu;
    if (!gate_open(a, DIRECT)) return;
    // the warps' stages in dynamic shared memory: double-buffered for the
    // stage kernel's cp.async prefetch, one per warp for the direct refill
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    WarpStage(*stages)[2] = reinterpret_cast<WarpStage(*)[2]>(dyn_smem);
    __shared__ unsigned shc[SC_N];
    __shared__ uint64_t sdig[THREADS];
    __shared__ int scnt[THREADS];
    VSLOTS_DECL(THREADS)
    counters_init(shc);
    const DigestSlot DS{sdig + threadIdx.x, scnt + threadIdx.x};
    const int wid = threadIdx.x >> 5;
    const int64_t nwork = DIRECT ? 0 : *nwork_p;
    auto claim = [&](WarpStage& st) -> int {
        return DIRECT ? claim_direct(a, D, st) : claim_chunk(a, W, st, nwork);
    };
    Lane L;
    L.busy = false;
    VSLOTS_INIT(L);
    Counters C;
    C.sh = shc;
    Pending P;
    P.init(a);
    int cur = 0;
    int head = 0;
    // direct refill: claim_direct's loads block anyway, so one stage per warp
    // (claimed when the previous one is used up) -- the second buffer's
    // shared memory goes to L1
    WarpStage* const st1 = reinterpret_cast<WarpStage*>(dyn_smem) + wid;
    int ncur = DIRECT ? claim(*st1) : claim(stages[wid][0]);
    int nnext = (!DIRECT && ncur == STAGE_N) ? claim(stages[wid][1]) : 0;
    // only the first group must have landed; wait_group 1 would do, but the
    // second claim may be empty -- a full wait costs one DRAM latency once
    cp_async_wait_all();
    __syncwarp();
    while (true) {
        unsigned idle = __ballot_sync(FULL, !L.busy);
        // Refill only once two lanes are idle (or none is busy): the refill is a
        // warp-wide detour, so serving two lanes per detour halves its cost for
        // a step of idleness per refill (-2..3% on the C2/C4/C5 walks; +4% on
        // a point source with long flights, whose lanes then start in pairs
        // from the same elements and collide in the tally atomics).
        if (__popc(idle) < REFILL_MIN && idle != FULL) idle = 0;
        while (idle) {
            if (head == ncur) {  // current stage used up: switch to the prefetched one
                if (DIRECT) {
                    if (ncur < STAGE_N) break;  // the last chunk was partial: no more work
                    __syncwarp();               // every lane is done reading the stage
                    ncur = claim(*st1);
                    head = 0;
                    if (ncur == 0) break;
                } else {
                    if (nnext == 0) break;
                    cp_async_wait_all();
                    __syncwarp();
                    cur ^= 1;
                    head = 0;
                    ncur = nnext;
                    // the stage just emptied is free: prefetch the chunk after next
                    nnext = (ncur == STAGE_N) ? claim(stages[wid][cur ^ 1]) : 0;
                }
            }
            const int take = min((int)__popc(idle), ncur - head);
            if (!L.busy) {
                const int rk = __popc(idle & lanemask_lt());
                const WarpStage& s = DIRECT ? *st1 : stages[wid][cur];
                const int j = head + rk;
                const int fl0 = rk < take ? s.fl[j] : 0;
                if (DIRECT && rk < take && !(fl0 & (1 << 24))) {
                    // not walked: a non-flying particle (empty digest) or a flying
                    // one that was never localized (counted, reported by the move)
                    if (fl0 & (1 << 25)) {
                        atomicAdd(a.counters + C_UNLOC, 1ull);
                    } else if (DIG && a.digest) {
                        a.digest[s.idx[j]] = DIGEST_INIT;
                        a.dcount[s.idx[j]] = 0;
                    }
                } else if (rk < take) {
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
                    vslots_fill(a, L, L.e, s.r0[j]);
                }
            }
            head += take;
            idle = __ballot_sync(FULL, !L.busy);
        }
        if (idle == FULL) {  // no work left anywhere for this warp (idle is current here)
            flush_pending(a, P, true);
            break;
        }
        if (L.busy) {
            if (walk_step<DIG>(a, L, C, P, DS)) finish<DIG>(a, L, C, DS);
        }
        // (a finished lane's pending score is issued by its next walk_step,
        // after the refill, or by the flush at the loop's exit: no idle flush)
        flush_pending(a, P, false);
    }
    cp_async_wait_all();
    flush_counters(a, C);
}

// Compact this move's flying particles into the work arrays (order of
// indices within a warp preserved; warps in arbitrary order).  Non-flying
// particles get an empty digest.
// Particles [lo, lo + a.count) of this move; work items go to W (already
// offset by the caller).  A flying particle with element < 0 is not staged
// and counted (the move then reports it).
__global__ void stage_kernel(const WalkArgs a, const WorkSoA W, int64_t* __restrict__ nwork,
                             int64_t lo) {
    if (!gate_open(a, false)) return;
    const int lane = threadIdx.x & 31;
    // grid-stride over warps (a bounded grid: when the device-side refill
    // choice gates this launch off, few CTAs have to start and return)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t wb = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); wb < a.count;
         wb += stride) {
        const int64_t t = wb + lane;
        bool fly = false;
        int64_t i = 0;
        if (t < a.count) {
            i = a.order ? (int64_t)a.order[t] : lo + t;
            fly = a.fly_in[i] != 0;
            if (a.digest && !fly) {
                a.digest[i] = DIGEST_INIT;
                a.dcount[i] = 0;
            }
            if (fly && a.element[i] < 0) {
                atomicAdd(a.counters + C_UNLOC, 1ull);
                fly = false;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, fly);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd((unsigned long long*)nwork, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (!fly) continue;
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
    }
}
