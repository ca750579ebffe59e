// move_prep.cuh -- move preparation, finalize, element-ordered hand-out keys.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

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
