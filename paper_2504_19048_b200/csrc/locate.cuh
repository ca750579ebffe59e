// locate.cuh -- localization: uniform grid, barycentric pre-filter records, grid search, walk-mode tie-break.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

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
    int prune;              // list elements only in cells their half-spaces reach
};

__device__ __forceinline__ int grid_axis(double p, double org, double cs, int dim) {
    double f = floor((p - org) / cs);
    int i = (f < 0.0) ? 0 : (f >= (double)dim ? dim - 1 : (int)f);
    return i;
}

// Which grid cells an element is listed in: the cells of its bounding box
// (expanded by 1e-7 of its extent) that its tolerance-expanded barycentric
// half-spaces do not exclude.  lambda_k is affine, so its maximum over a cell
// is w_k.(c - v0) + |w_k|.h (c the centre, h the half-size): a cell where one
// maximum is below -CELL_TOL cannot hold a point the element contains
// (the reference's containment tolerance is EPS_BARY = 1e-10 plus its own
// rounding, <= 1e-8 for the elements this test applies to: quality ratio
// A^3/|det| <= 1e6; others keep every box cell).  A Kuhn tet fills a sixth of
// its box: the cells' candidate lists shrink ~2.5x, and the lowest-id search
// scans half a list per point.
constexpr double CELL_TOL = 1e-6;
struct ElemCells {
    int lo[3], hi[3];  // cell index range of the expanded box
    double w[4][3];    // lambda_k = w_k . (p - v0) (+ 1 for k = 0)
    double v0[3];
    bool prune;        // false: keep every box cell
};
__device__ inline ElemCells elem_cells(const ElemRec& r, const Vtx* __restrict__ vtx,
                                       const GridDev& G) {
    ElemCells E;
    double x[4], y[4], z[4];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int j = 0; j < 4; ++j) {
        const Vtx v = vtx[r.v[j]];
        x[j] = v.x;
        y[j] = v.y;
        z[j] = v.z;
        const double c[3] = {v.x, v.y, v.z};
        for (int k = 0; k < 3; ++k) {
            lo[k] = fmin(lo[k], c[k]);
            hi[k] = fmax(hi[k], c[k]);
        }
    }
    const double ext = fmax(fmax(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
    const double delta = 1e-7 * ext + 1e-300;
    for (int k = 0; k < 3; ++k) {
        E.lo[k] = grid_axis(lo[k] - delta, G.org[k], G.cs[k], G.dims[k]);
        E.hi[k] = grid_axis(hi[k] + delta, G.org[k], G.cs[k], G.dims[k]);
    }
    double a[3][3];
    for (int k = 0; k < 3; ++k) {
        a[k][0] = x[k + 1] - x[0];
        a[k][1] = y[k + 1] - y[0];
        a[k][2] = z[k + 1] - z[0];
    }
    double n[3][3];
    auto cross = [](const double* u, const double* v, double* o) {
        o[0] = u[1] * v[2] - u[2] * v[1];
        o[1] = u[2] * v[0] - u[0] * v[2];
        o[2] = u[0] * v[1] - u[1] * v[0];
    };
    cross(a[1], a[2], n[0]);
    cross(a[2], a[0], n[1]);
    cross(a[0], a[1], n[2]);
    const double det = a[0][0] * n[0][0] + a[0][1] * n[0][1] + a[0][2] * n[0][2];
    double A = 0.0;
    for (int k = 0; k < 3; ++k) A = fmax(A, fabs(a[k][0]) + fabs(a[k][1]) + fabs(a[k][2]));
    const double q = A * A * A / fabs(det);
    E.prune = G.prune && q <= 1e6;  // false for NaN / inf (degenerate elements)
    for (int i = 0; i < 3; ++i) E.w[0][i] = 0.0;
    for (int k = 0; k < 3; ++k)
        for (int i = 0; i < 3; ++i) {
            E.w[k + 1][i] = n[k][i] / det;
            E.w[0][i] -= E.w[k + 1][i];
        }
    E.v0[0] = x[0];
    E.v0[1] = y[0];
    E.v0[2] = z[0];
    return E;
}
__device__ inline bool elem_cell_overlap(const ElemCells& E, const GridDev& G, int i, int j,
                                         int l) {
    if (!E.prune) return true;
    const int ix[3] = {i, j, l};
    double d[3], h[3];
    for (int k = 0; k < 3; ++k) {
        h[k] = 0.5 * G.cs[k] * (1.0 + 2e-7);  // the point-to-cell mapping's rounding
        d[k] = G.org[k] + ((double)ix[k] + 0.5) * G.cs[k] - E.v0[k];
    }
    for (int k = 0; k < 4; ++k) {
        const double lmax = (k == 0 ? 1.0 : 0.0) + E.w[k][0] * d[0] + E.w[k][1] * d[1] +
                            E.w[k][2] * d[2] +
                            (fabs(E.w[k][0]) * h[0] + fabs(E.w[k][1]) * h[1] + fabs(E.w[k][2]) * h[2]);
        if (lmax < -CELL_TOL) return false;  // the whole cell is beyond face k
    }
    return true;
}

__global__ void elem_cells_count_kernel(const ElemRec* __restrict__ rec,
                                        const Vtx* __restrict__ vtx, int64_t ne, GridDev G,
                                        long long* __restrict__ counts) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const ElemCells E = elem_cells(rec[e], vtx, G);
    int cnt = 0;
    for (int i = E.lo[0]; i <= E.hi[0]; ++i)
        for (int j = E.lo[1]; j <= E.hi[1]; ++j)
            for (int l = E.lo[2]; l <= E.hi[2]; ++l) cnt += elem_cell_overlap(E, G, i, j, l);
    counts[e] = cnt;
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

__global__ void elem_cells_emit_kernel(int64_t ne, GridDev G, const ElemRec* __restrict__ rec,
                                       const Vtx* __restrict__ vtx, const long long* __restrict__ offs,
                                       unsigned long long* __restrict__ keys) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const ElemCells E = elem_cells(rec[e], vtx, G);  // the same decisions as the count
    long long k = offs[e];
    for (int i = E.lo[0]; i <= E.hi[0]; ++i)
        for (int j = E.lo[1]; j <= E.hi[1]; ++j)
            for (int l = E.lo[2]; l <= E.hi[2]; ++l)
                if (elem_cell_overlap(E, G, i, j, l)) {
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
    int32_t exact_only;  // BT_OPT_EXACT_ONLY: every candidate takes the exact test
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
            const int pre = a.exact_only ? 0 : lambda_prefilter(a.lam + c, q0, q1, q2);
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
