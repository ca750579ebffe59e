// Host self-test of the filtered exit search (csrc/geometry.cuh): walks
// particles through a mesh on the CPU, and at EVERY step compares
// exit_search_fast() against exit_search() (the reference's literal
// arithmetic), following the literal result.  Built by
// tests/test_filter_selftest.py with nvcc (host code, -ffp-contract=off).
#include <cstdint>
#include <cstring>

#include "../../paper_2504_19048_b200/csrc/geometry.cuh"

using namespace bt;

// The round-1 scalar formulation of exit_filter32 (one fp32 operation per
// instruction): the packed filter in geometry.cuh must return the same
// decisions and the same probed intermediates, bit for bit.
static int exit_filter32_scalar(const Tet& T, double ox, double oy, double oz, double dx, double dy,
                        double dz, int entry, int* face, unsigned* qmask, int* why = nullptr,
                        F32Probe* probe = nullptr) {
    const double x0 = T.x[0], y0 = T.y[0], z0 = T.z[0];
    const float a1x = f32(T.x[1] - x0), a1y = f32(T.y[1] - y0), a1z = f32(T.z[1] - z0);
    const float a2x = f32(T.x[2] - x0), a2y = f32(T.y[2] - y0), a2z = f32(T.z[2] - z0);
    const float a3x = f32(T.x[3] - x0), a3y = f32(T.y[3] - y0), a3z = f32(T.z[3] - z0);
    const float sx = f32(rn_sub(dx, ox)), sy = f32(rn_sub(dy, oy)), sz = f32(rn_sub(dz, oz));
    const float r0x = f32(x0 - ox), r0y = f32(y0 - oy), r0z = f32(z0 - oz);
    const float g2x = fsub(a1x, a2x), g2y = fsub(a1y, a2y), g2z = fsub(a1z, a2z);
    const float g3x = fsub(a1x, a3x), g3y = fsub(a1y, a3y), g3z = fsub(a1z, a3z);
    const float r1x = fadd(a1x, r0x), r1y = fadd(a1y, r0y), r1z = fadd(a1z, r0z);
    const float S = n1f(sx, sy, sz);
    const float Nx = std::fmax(
        std::fmax(std::fmax(n1f(a1x, a1y, a1z), n1f(a2x, a2y, a2z)),
                  std::fmax(n1f(a3x, a3y, a3z), n1f(g2x, g2y, g2z))),
        std::fmax(n1f(g3x, g3y, g3z), std::fmax(n1f(r0x, r0y, r0z), n1f(r1x, r1y, r1z))));
    // every early-out is decided at the end instead: a data-dependent branch
    // in mid-filter stops the warp (in-order issue) until its chain resolves,
    // while the rest of the filter does not depend on it.  Results identical.
    const bool range_ok = (Nx >= 1e-10f) & (Nx <= 1e10f) & (S <= 1e10f);
    const float N2 = fmul(Nx, Nx);
    const float n1x = crf(a2y, a3z, a2z, a3y), n1y = crf(a2z, a3x, a2x, a3z),
                n1z = crf(a2x, a3y, a2y, a3x);
    const float n2x = crf(a1y, a3z, a1z, a3y), n2y = crf(a1z, a3x, a1x, a3z),
                n2z = crf(a1x, a3y, a1y, a3x);
    const float n3x = crf(a1y, a2z, a1z, a2y), n3y = crf(a1z, a2x, a1x, a2z),
                n3z = crf(a1x, a2y, a1y, a2x);
    // Destination containment from the face determinants: with b = d - v0 =
    // s - r0, the reference's numerators are b.n_k = D_k - NT_k (k = 1..3) and
    // |Dc| - t1 - t2 - t3 = sign(Dc) (NT0 - D0) (since n0 = n1 - n2 + n3 and
    // a1.n0 = Dc), so the four quantities cost one subtraction each.  Each is
    // within 14.1 + 14.1 + 1.01 = 29.3 u P32 <= 37 u Pc of its exact value.
    const float Dc = dtf(a1x, a1y, a1z, n1x, n1y, n1z);
    const float Mc = MC32_REL * fmul(N2, ffm(2.0f, Nx, S));
    const float aDc = std::fabs(Dc);
    const bool dc_ok = aDc > Mc;
    bool pass, fail;
    // D_f = s.n_f, NT_f = r.n_f
    const float D1 = dtf(sx, sy, sz, n1x, n1y, n1z), NT1 = dtf(r0x, r0y, r0z, n1x, n1y, n1z);
    const float D2 = dtf(sx, sy, sz, n2x, n2y, n2z), NT2 = dtf(r0x, r0y, r0z, n2x, n2y, n2z);
    const float D3 = dtf(sx, sy, sz, n3x, n3y, n3z), NT3 = dtf(r0x, r0y, r0z, n3x, n3y, n3z);
    const float n0x = crf(g2y, g3z, g2z, g3y), n0y = crf(g2z, g3x, g2x, g3z),
                n0z = crf(g2x, g3y, g2y, g3x);
    const float D0 = dtf(sx, sy, sz, n0x, n0y, n0z), NT0 = dtf(r1x, r1y, r1z, n0x, n0y, n0z);
    const float P32 = fmul(N2, fadd(S, Nx));
    {
        const float t1 = flip_byf(fsub(D1, NT1), Dc);
        const float t2 = flip_byf(fsub(NT2, D2), Dc);
        const float t3 = flip_byf(fsub(D3, NT3), Dc);
        const float y0s = flip_byf(fsub(NT0, D0), Dc);
        if (probe && range_ok && dc_ok) {
            probe->stage = 1;
            probe->S = S;
            probe->Nx = Nx;
            probe->Dc = Dc;
            probe->t[0] = t1;
            probe->t[1] = t2;
            probe->t[2] = t3;
            probe->y0 = y0s;
            probe->Pc = fmul(N2, ffm(2.0f, Nx, S));
            probe->P32 = P32;
        }
        const float tolD = fmul((float)EPS_BARY, aDc);
        const float hi = fsub(Mc, tolD), lo = fsub(-Mc, tolD);
        fail = (t1 < lo) | (t2 < lo) | (t3 < lo) | (y0s < lo);
        pass = (t1 > hi) & (t2 > hi) & (t3 > hi) & (y0s > hi);
    }
    const float M = M16_REL * P32;
    // k1 = M16 / M1 = (S + Nx) / (Nx + 1e-12 S)
#if defined(__CUDA_ARCH__)
    // approximate division (<= 2 ulp, 2.4e-7 relative): k1 only scales x1,
    // far inside the 5% slack of its margin
    const float k1 = __fdividef(fadd(S, Nx), ffm(1e-12f, S, Nx));
#else
    const float k1 = fadd(S, Nx) / ffm(1e-12f, S, Nx);
#endif
    const float m0x = crf(sy, r0z, sz, r0y), m0y = crf(sz, r0x, sx, r0z), m0z = crf(sx, r0y, sy, r0x);
    const float p1 = dtf(a1x, a1y, a1z, m0x, m0y, m0z);
    const float p2 = dtf(a2x, a2y, a2z, m0x, m0y, m0z);
    const float p3 = dtf(a3x, a3y, a3z, m0x, m0y, m0z);
    // NU_f = e2.m, NW_f = -(e1.m)
    const float m1x = crf(sy, r1z, sz, r1y), m1y = crf(sz, r1x, sx, r1z),
                m1z = crf(sx, r1y, sy, r1x);
    const float NU0 = dtf(g3x, g3y, g3z, m1x, m1y, m1z), NW0 = -dtf(g2x, g2y, g2z, m1x, m1y, m1z);
    if (probe && range_ok && dc_ok && !pass && fail) {
        probe->stage = 2;
        const float d[4] = {D0, D1, D2, D3}, nt[4] = {NT0, NT1, NT2, NT3};
        const float nu[4] = {NU0, -p3, -p3, -p2}, nw[4] = {NW0, p2, p1, p1};
        for (int f = 0; f < 4; ++f) {
            probe->D[f] = d[f];
            probe->NT[f] = nt[f];
            probe->NU[f] = nu[f];
            probe->NW[f] = nw[f];
        }
    }
    int st[4];
    st[1] = face_state32(D1, NT1, -p3, p2, M, k1);
    st[2] = face_state32(D2, NT2, -p3, p1, M, k1);
    st[3] = face_state32(D3, NT3, -p2, p1, M, k1);
    st[0] = face_state32(D0, NT0, NU0, NW0, M, k1);
    // face selection on bit masks (faces other than the entry face)
    const unsigned consider = entry >= 0 ? (0xFu & ~(1u << entry)) : 0xFu;
    const unsigned pm = (unsigned)(st[0] > 0) | ((unsigned)(st[1] > 0) << 1) |
                        ((unsigned)(st[2] > 0) << 2) | ((unsigned)(st[3] > 0) << 3);
    const unsigned um = (unsigned)(st[0] == 0) | ((unsigned)(st[1] == 0) << 1) |
                        ((unsigned)(st[2] == 0) << 2) | ((unsigned)(st[3] == 0) << 3);
    const unsigned qm = pm & consider;
    if (!range_ok) {
        if (why) *why = 1;
        return XF_EXACT;
    }
    if (!dc_ok) {
        if (why) *why = 2;
        return XF_EXACT;
    }
    if (pass) return XF_REACHED;
    if (!fail) {
        if (why) *why = 3;
        return XF_EXACT;
    }
    if ((um & consider) || !qm) {
        if (why) *why = (um & consider) ? 4 : 5;
        return XF_EXACT;
    }
    *face = bt_ctz(qm);
    *qmask = qm;
    return (qm & (qm - 1)) == 0 ? XF_EXIT : XF_MULTI;
}



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
                int w3 = 0;
                const int x3 = exit_filter32(T, ox, oy, oz, dx, dy, dz, entry, &f3, &q3, &w3);
                if (x3 == XF_EXACT) ++und32;
                // packed (FFMA2) filter == the scalar formulation, decision for decision
                int f5 = -1, w5 = 0;
                unsigned q5 = 0;
                const int x5 = exit_filter32_scalar(T, ox, oy, oz, dx, dy, dz, entry, &f5, &q5, &w5);
                if (x3 != x5 || w3 != w5 || (x3 != XF_EXACT && (f3 != f5 || q3 != q5))) ++mism;
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
                             const double* od /* 6 per case */, int64_t n, float* out,
                             int64_t* packed_mismatch) {
    *packed_mismatch = 0;
    for (int64_t i = 0; i < n; ++i) {
        Tet T;
        for (int j = 0; j < 4; ++j) {
            T.x[j] = tets[12 * i + j];
            T.y[j] = tets[12 * i + 4 + j];
            T.z[j] = tets[12 * i + 8 + j];
        }
        F32Probe p{}, ps{};
        int f = -1, fs = -1;
        unsigned q = 0, qs = 0;
        const int x = exit_filter32(T, od[6 * i], od[6 * i + 1], od[6 * i + 2], od[6 * i + 3],
                                    od[6 * i + 4], od[6 * i + 5], -1, &f, &q, nullptr, &p);
        const int xs = exit_filter32_scalar(T, od[6 * i], od[6 * i + 1], od[6 * i + 2],
                                            od[6 * i + 3], od[6 * i + 4], od[6 * i + 5], -1, &fs,
                                            &qs, nullptr, &ps);
        // the packed filter's intermediates equal the scalar formulation's
        // (== on floats: a negated exact difference may carry the other zero sign)
        bool same = x == xs && p.stage == ps.stage;
        if (same && p.stage >= 1) {
            same = p.S == ps.S && p.Nx == ps.Nx && p.Dc == ps.Dc && p.y0 == ps.y0 &&
                   p.Pc == ps.Pc && p.P32 == ps.P32;
            for (int k = 0; k < 3; ++k) same = same && p.t[k] == ps.t[k];
        }
        if (same && p.stage == 2)
            for (int k = 0; k < 4; ++k)
                same = same && p.D[k] == ps.D[k] && p.NT[k] == ps.NT[k] && p.NU[k] == ps.NU[k] &&
                       p.NW[k] == ps.NW[k];
        if (!same) ++*packed_mismatch;
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
