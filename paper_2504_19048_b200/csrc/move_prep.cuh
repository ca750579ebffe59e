// move_prep.cuh -- move preparation, finalize, element-ordered hand-out keys.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

// ---------------------------------------------------------------------------
// move preparation (device-resident inputs): group range check; flags bit 1
// = a flying particle is not localized, bit 2 = a group id outside
// [0, ngroups) (the move's walk kernels then do nothing: MoveGate)

__global__ void prepare_kernel(const int8_t* __restrict__ fly, const int32_t* __restrict__ element,
                               const int32_t* __restrict__ groups, int32_t ngroups, int64_t count,
                               unsigned long long* __restrict__ flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool unloc = false, badg = false;
    if (i < count) {
        const bool f = fly[i] != 0;
        unloc = f && element[i] < 0;
        if (groups) badg = groups[i] < 0 || groups[i] >= ngroups;
    }
    if (__any_sync(0xffffffffu, unloc) && (threadIdx.x & 31) == 0) atomicOr(flags, 1ull);
    if (__any_sync(0xffffffffu, badg) && (threadIdx.x & 31) == 0) atomicOr(flags, 2ull);
}

// ---------------------------------------------------------------------------
// Recorded source weight of a device-input move: numpy's pairwise summation
// (numpy/_core/src/umath/loops_utils.h.src, pairwise_sum_DOUBLE) of the
// flying particles' weights in index order -- the reference's
// `weight[:count][fly.astype(bool)].sum()` (tally.py:267-269) bit for bit,
// and the same value the host-input path computes (b200tally.cu
// pairwise_sum).  The selection is compacted first (CUB DeviceSelect); the
// summation tree is then evaluated with one thread per leaf (<= 128 values,
// eight accumulators as numpy) and the inner nodes by the second of the two
// children to finish (ticket per node, reset on use), so the association is
// numpy's whatever the scheduling.

__device__ __forceinline__ double pairwise_leaf(const double* __restrict__ a, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[i + k]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// Thread t follows the bits of t (most significant first) from the root of
// the tree over [0, *m); the first node of <= 128 values on its path is a
// leaf, summed by the thread whose remaining bits are zero.  `depth` is
// chosen by the host so that every node at that depth is a leaf
// (capacity / 2^depth <= 64 gives nodes of <= 80 values).  vals/ticks are
// heap-indexed (root 1) with 2^(depth+1) entries; ticks start (and end) 0.
__global__ void pairwise_sum_kernel(const double* __restrict__ a,
                                    const long long* __restrict__ m_p, int depth,
                                    double* __restrict__ vals, unsigned* __restrict__ ticks,
                                    double* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t(1) << depth)) return;
    int64_t lo = 0, n = *m_p;
    int64_t node = 1;
    int d = 0;
    while (n > 128) {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        const int bit = (int)((t >> (depth - 1 - d)) & 1);
        if (bit) {
            lo += n2;
            n -= n2;
        } else {
            n = n2;
        }
        node = 2 * node + bit;
        ++d;
    }
    if (d < depth && (t & ((int64_t(1) << (depth - d)) - 1)) != 0) return;  // not the representative
    double v = pairwise_leaf(a + lo, n);
    while (node > 1) {
        vals[node] = v;
        __threadfence();
        const int64_t p = node >> 1;
        if (atomicAdd(ticks + p, 1u) == 0) return;  // the sibling finishes the parent
        ticks[p] = 0;
        __threadfence();
        const double other = *(volatile double*)(vals + (node ^ 1));
        v = (node & 1) ? __dadd_rn(other, v) : __dadd_rn(v, other);
        node = p;
    }
    *out = v;
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

// walkable particles of a move (flying and localized): picks the refill mode
__global__ void count_walkable_kernel(const int8_t* __restrict__ fly,
                                      const int32_t* __restrict__ element, int64_t n,
                                      unsigned long long* __restrict__ out) {
    unsigned c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        c += fly[i] != 0 && element[i] >= 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// crossing records (layout.cuh XRec): the new vertex and the
// vertex-order selector of every face's neighbour; *bad counts faces whose
// neighbour does not share the face's three vertices (non-conforming mesh)
__global__ void xrec_kernel(const ElemRec* __restrict__ rec, int64_t ne, XRec* __restrict__ xrec,
                            unsigned* __restrict__ xsel /* null: pack into nvs */,
                            unsigned long long* bad) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const ElemRec r = rec[e];
    XRec x;
    unsigned sel[4];
    for (int f = 0; f < 4; ++f) {
        x.nbp[f] = r.nb[f];
        x.nvs[f] = 0;
        sel[f] = 0;
        if (r.nb[f] < 0) continue;
        const ElemRec q = rec[r.nb[f] >> 2];
        const int nf = r.nb[f] & 3;
        x.nvs[f] = (unsigned)q.v[nf];
        for (int k = 0; k < 4; ++k) {
            int j = f;  // slot of the leaving vertex receives the new one
            if (k != nf) {
                j = -1;
                for (int i = 0; i < 4; ++i)
                    if (i != f && r.v[i] == q.v[k]) j = i;
                if (j < 0) {
                    atomicAdd(bad, 1ull);
                    j = 0;
                }
            }
            sel[f] |= (unsigned)j << (2 * k);
        }
        if (!xsel) x.nvs[f] |= sel[f] << 24;
    }
    xrec[e] = x;
    if (xsel) xsel[e] = sel[0] | (sel[1] << 8) | (sel[2] << 16) | (sel[3] << 24);
}
