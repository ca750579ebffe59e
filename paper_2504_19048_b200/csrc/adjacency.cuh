// adjacency.cuh -- GPU mesh ingest: face adjacency by radix sorts.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

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
