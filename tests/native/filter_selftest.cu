// Host self-test of the filtered exit search (csrc/geometry.cuh): walks
// particles through a mesh on the CPU, and at EVERY step compares
// exit_search_fast() against exit_search() (the reference's literal
// arithmetic), following the literal result.  Built by
// tests/test_filter_selftest.py with nvcc (host code, -ffp-contract=off).
#include <cstdint>
#include <cstring>

#include "../../paper_2504_19048_b200/csrc/geometry.cuh"

using namespace bt;

extern "C" int bt_filter_selftest(const double* vertices, const int32_t* elements,
                                  const int32_t* adj_elem, const int8_t* adj_face,
                                  const int32_t* start_elem, const double* start_pos,
                                  const double* dest, int64_t n, int64_t max_steps,
                                  int64_t* stats /* steps, mismatches, fallbacks, stuck,
                                                    fp32-undecided */) {
    int64_t steps = 0, mism = 0, fb = 0, stuck = 0, und32 = 0;
    for (int64_t i = 0; i < n; ++i) {
        int e = start_elem[i];
        if (e < 0) continue;
        double ox = start_pos[3 * i], oy = start_pos[3 * i + 1], oz = start_pos[3 * i + 2];
        const double dx = dest[3 * i], dy = dest[3 * i + 1], dz = dest[3 * i + 2];
        int entry = -1;
        for (int64_t k = 0; k < max_steps; ++k) {
            Tet T;
            for (int j = 0; j < 4; ++j) {
                const int v = elements[4 * e + j];
                T.x[j] = vertices[3 * v];
                T.y[j] = vertices[3 * v + 1];
                T.z[j] = vertices[3 * v + 2];
            }
            int f1 = 0, f2 = 0;
            double t1 = 0, t2 = 0;
            bool ex = false;
            const int k1 = exit_search(T, ox, oy, oz, dx, dy, dz, entry, &f1, &t1);
            const int k2 = exit_search_fast(T, ox, oy, oz, dx, dy, dz, entry, &f2, &t2, &ex);
            ++steps;
            if (ex) ++fb;
            {
                int f3 = -1;
                unsigned q3 = 0;
                if (exit_filter32(T, ox, oy, oz, dx, dy, dz, entry, &f3, &q3) == XF_EXACT) ++und32;
                // the fp64 filter (BT_F64_STAGE builds) against the literal result
                int f4 = -1;
                unsigned q4 = 0;
                const int x4 = exit_filter(T, ox, oy, oz, dx, dy, dz, entry, &f4, &q4);
                if ((x4 == XF_REACHED && k1 != 0) || (x4 == XF_EXIT && (k1 != 1 || f4 != f1)) ||
                    (x4 == XF_MULTI && (k1 != 1 || !((q4 >> f1) & 1u))))
                    ++mism;
            }
            if (k1 != k2 || f1 != f2 || std::memcmp(&t1, &t2, sizeof t1) != 0) ++mism;
            if (k1 != 1) {
                if (k1 == 2) ++stuck;
                break;
            }
            const double qx = rn_add(ox, rn_mul(t1, rn_sub(dx, ox)));
            const double qy = rn_add(oy, rn_mul(t1, rn_sub(dy, oy)));
            const double qz = rn_add(oz, rn_mul(t1, rn_sub(dz, oz)));
            const int nb = adj_elem[4 * e + f1];
            if (nb < 0) break;
            entry = adj_face[4 * e + f1];
            e = nb;
            ox = qx;
            oy = qy;
            oz = qz;
        }
    }
    stats[0] = steps;
    stats[1] = mism;
    stats[2] = fb;
    stats[3] = stuck;
    stats[4] = und32;
    return 0;
}

// contains_fast() vs contains() for every (point, element) pair.
extern "C" int64_t bt_contains_selftest(const double* vertices, const int32_t* elements,
                                        int64_t ne, const double* pts, int64_t n, double tol,
                                        int64_t* fallbacks) {
    int64_t mism = 0, fb = 0;
    for (int64_t e = 0; e < ne; ++e) {
        Tet T;
        for (int j = 0; j < 4; ++j) {
            const int v = elements[4 * e + j];
            T.x[j] = vertices[3 * v];
            T.y[j] = vertices[3 * v + 1];
            T.z[j] = vertices[3 * v + 2];
        }
        for (int64_t i = 0; i < n; ++i) {
            const bool a = contains(T, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], tol);
            const bool b = contains_fast(T, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], tol);
            if (a != b) ++mism;
        }
    }
    *fallbacks = fb;
    return mism;
}

// The fp32 filter's intermediate quantities for n (tet, origin, destination)
// cases: out[27*i ...] = stage, S, R0(unused), Nx, Dc, t1..t3, y0, Pc, P32,
// D[4], NT[4], NU[4], NW[4] (tests/test_filter_bounds.py checks them against
// exact rational determinants of the reference's fp64 vectors).
extern "C" void bt_f32_probe(const double* tets /* 12 per case: x0..3, y0..3, z0..3 */,
                             const double* od /* 6 per case */, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) {
        Tet T;
        for (int j = 0; j < 4; ++j) {
            T.x[j] = tets[12 * i + j];
            T.y[j] = tets[12 * i + 4 + j];
            T.z[j] = tets[12 * i + 8 + j];
        }
        F32Probe p{};
        int f = -1;
        unsigned q = 0;
        exit_filter32(T, od[6 * i], od[6 * i + 1], od[6 * i + 2], od[6 * i + 3], od[6 * i + 4],
                      od[6 * i + 5], -1, &f, &q, nullptr, &p);
        float* o = out + 27 * i;
        const float head[11] = {(float)p.stage, p.S, p.R0, p.Nx, p.Dc, p.t[0], p.t[1], p.t[2],
                                p.y0, p.Pc, p.P32};
        for (int k = 0; k < 11; ++k) o[k] = head[k];
        for (int k = 0; k < 4; ++k) {
            o[11 + k] = p.D[k];
            o[15 + k] = p.NT[k];
            o[19 + k] = p.NU[k];
            o[23 + k] = p.NW[k];
        }
    }
}
