// layout.cuh -- device data layout of the walk: element records, vertices, walk arguments, loads.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

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

// Crossing record: per face f of an element, the neighbour
// across f ((nb << 2) | nf, -1 on the boundary) and the one vertex of the
// neighbour that is not on f (its local vertex nf).  The other three are
// the element's own, so a crossing fetches ONE vertex, at the same time as
// the neighbour's record, instead of record -> four vertices.  sel[f] maps
// the neighbour's local vertex order onto the element's: bits 2k..2k+1 =
// the element's local index of the neighbour's vertex k (f itself for
// k = nf, whose slot receives the new vertex).  nvs[f] = nv | sel << 24 in
// one 32-byte sector; meshes of 2^24 vertices or more keep nv whole and the
// four sel bytes in a separate array (WalkArgs::xsel, one more sector).
struct __align__(16) XRec {
    int nbp[4];
    unsigned nvs[4];
};
static_assert(sizeof(XRec) == 32, "one 32-byte sector per element");

enum { C_EVENTS = 0, C_REACHED, C_BOUNDARY, C_RECOV, C_KILLED, C_SWEEPS, C_ERR, C_UNLOC, C_NCOUNTERS };
// dcounters layout (unsigned long long): [1..8] counters, [9] the recorded
// source weight of a device-input move (double bits), [10] its selected
// count, [14] walkable count (refill choice), [15] flags,
// [16 + c] queue of chunk c, [32 + c] work count of chunk c, c < MAX_CHUNKS
constexpr int MAX_CHUNKS = 16;
constexpr int DC_SOURCE_WEIGHT = 9, DC_SELECTED = 10;
constexpr int NDCOUNTERS = 48;

// __match_any_sync aggregation of the tally atomics (BT_OPT_WARP_AGG)
enum { WAGG_ADAPTIVE = 0, WAGG_ALWAYS = 1, WAGG_NEVER = 2 };

struct WalkArgs {
    const ElemRec* __restrict__ rec;
    const Vtx* __restrict__ vtx;
    const XRec* __restrict__ xrec;       // (E) crossing records
    const unsigned* __restrict__ xsel;   // (E) sel[4] as 4 bytes; null: packed in nvs
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
    int32_t exact_only;  // digest kernels only: literal exit search (filter validation)
    // Device-side decision of a move (nullable): gate[0] = walkable particles
    // of the move, gate[1] = prepare_kernel's flags.  Every walk launch of the
    // move returns at once when flags bit 2 is set (a group out of range: the
    // move fails before any work); with gate_pick, the direct-refill walk runs
    // iff 2 * walkable >= count and the stage-kernel pair otherwise (both are
    // enqueued; the other returns at once), so the host never waits for the
    // choice.
    const unsigned long long* gate;
    int32_t gate_pick;
    // Host-input move streamed into one direct-refill launch (nullable): the
    // particles below *ready have landed; a warp claiming beyond it waits.
    // Written by the copy stream (a stream memory operation after each chunk's
    // copies), so the walk starts after the first chunk, not the last.
    const unsigned long long* ready;
};

// the launch runs (see WalkArgs::gate); DIRECT: the direct-refill walk
__device__ __forceinline__ bool gate_open(const WalkArgs& a, bool direct) {
    if (!a.gate) return true;
    const unsigned long long walkable = a.gate[0], flags = a.gate[1];
    if (flags & 2ull) return false;
    return !a.gate_pick || ((2 * (long long)walkable >= a.count) == direct);
}

#ifndef BT_NO_L2_HINT
// Mesh gathers carry an L2 evict_last policy, so the streamed particle state
// and work list are evicted first (3% on the C2 walk, 0.7% when the mesh
// exceeds L2: tools/sweep.py --which c4 with -DBT_NO_L2_HINT as the control).
__device__ __forceinline__ unsigned long long mesh_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double2 ldg_mesh(const double2* p) {
    double2 v;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
        : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(mesh_policy()));
    return v;
}
__device__ __forceinline__ int4 ldg_mesh(const int4* p) {
    int4 v;
    asm("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(mesh_policy()));
    return v;
}
#else
__device__ __forceinline__ double2 ldg_mesh(const double2* p) { return __ldg(p); }
__device__ __forceinline__ int4 ldg_mesh(const int4* p) { return __ldg(p); }
#endif

__device__ __forceinline__ void load_tet(const WalkArgs& a, const ElemRec& r, Tet& T) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double2* p = reinterpret_cast<const double2*>(a.vtx + r.v[j]);
        const double2 xy = ldg_mesh(p);
        const double2 zw = ldg_mesh(p + 1);
        T.x[j] = xy.x;
        T.y[j] = xy.y;
        T.z[j] = zw.x;
    }
}

__device__ __forceinline__ ElemRec load_rec(const ElemRec* __restrict__ rec, int e) {
    const int4* p = reinterpret_cast<const int4*>(rec + e);
    const int4 a = ldg_mesh(p);
    const int4 b = ldg_mesh(p + 1);
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
