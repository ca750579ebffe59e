/*
 * walk_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs as the CHECKER and the CPU
 * baseline.  The product path (paper_2504_19048_b200, libb200tally.so) never
 * links or calls this file.
 *
 * Parity pin: checked against golden vectors produced by running the
 * reference itself (oracle/gen_golden.py writes the tests/golden fixtures), see
 * tests/test_oracle_golden.py.
 *
 * Arithmetic contract: IEEE fp64 with no
 * contraction (-ffp-contract=off), operands in the reference's order, true
 * divisions, sqrt.  numba compiles the reference without fastmath (0 FMA,
 * 3 divsd per solve), so these functions reproduce its bits.
 *
 * Sources restated (file:line in /root/reference/pkg/src/meshtally):
 *   det3                 geometry.py:49-53
 *   bary_core            geometry.py:56-73
 *   face_hit_core        geometry.py:93-114
 *   _FV0/_FV1/_FV2       geometry.py:117-120
 *   elem_contains        geometry.py:149-154
 *   exit_search_core     geometry.py:167-189
 *   _compact_flying      search.py:160-166
 *   _sweep_fused         search.py:169-275
 *   trace_and_score      search.py:492-517 (sweep guard 449-450)
 *   _tie_break_faces     search.py:520-551
 *   initialize_locations search.py:557-601
 *   _finalize            tally.py:83-95
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EPS_BARY 1e-10
#define EPS_T 1e-12
#define STUCK_TOL_FACTOR 10.0
#define NUDGE 1e-9

enum { OUT_NONE = 0, OUT_REACHED = 1, OUT_LEAKED = 2, OUT_STUCK_KILLED = 3 };

static const int FV0[4] = {1, 0, 0, 0};
static const int FV1[4] = {2, 2, 1, 1};
static const int FV2[4] = {3, 3, 3, 2};

#define DIGEST_INIT 0xcbf29ce484222325ULL
#define DIGEST_PRIME 0x100000001b3ULL

typedef struct {
    const double *vertices;   /* (V,3) */
    const int32_t *elements;  /* (E,4) */
    const int32_t *adj_elem;  /* (E,4) */
    const int8_t *adj_face;   /* (E,4) */
    int64_t num_elements;
} om_mesh;

typedef struct {
    double *position;          /* (N,3) */
    const double *destination; /* (N,3) */
    const double *weight;      /* (N)   */
    const int32_t *group;      /* (N)   */
    int32_t *element;
    int8_t *flying;
    int8_t *alive;
    int8_t *entry_face;
    int8_t *stuck;
    int8_t *outcome;
    double *seg_total;
    uint64_t *digest;          /* nullable: per-particle sequence digest */
    int64_t *count;            /* nullable: per-particle scored events */
} om_particles;

static inline double det3(double a11, double a12, double a13, double a21, double a22,
                          double a23, double a31, double a32, double a33) {
    return (a11 * (a22 * a33 - a23 * a32) - a12 * (a21 * a33 - a23 * a31)) +
           a13 * (a21 * a32 - a22 * a31);
}

/* returns d (6x signed volume); l[0..3] garbage when d == 0 */
static inline double bary_core(const double v[4][3], double px, double py, double pz,
                               double l[4]) {
    double a11 = v[1][0] - v[0][0], a21 = v[1][1] - v[0][1], a31 = v[1][2] - v[0][2];
    double a12 = v[2][0] - v[0][0], a22 = v[2][1] - v[0][1], a32 = v[2][2] - v[0][2];
    double a13 = v[3][0] - v[0][0], a23 = v[3][1] - v[0][1], a33 = v[3][2] - v[0][2];
    double bx = px - v[0][0], by = py - v[0][1], bz = pz - v[0][2];
    double d = det3(a11, a12, a13, a21, a22, a23, a31, a32, a33);
    if (d == 0.0) {
        l[0] = l[1] = l[2] = l[3] = 0.0;
        return 0.0;
    }
    double l1 = det3(bx, a12, a13, by, a22, a23, bz, a32, a33) / d;
    double l2 = det3(a11, bx, a13, a21, by, a23, a31, bz, a33) / d;
    double l3 = det3(a11, a12, bx, a21, a22, by, a31, a32, bz) / d;
    l[0] = ((1.0 - l1) - l2) - l3;
    l[1] = l1;
    l[2] = l2;
    l[3] = l3;
    return d;
}

static inline double face_hit_core(const double a[3], const double b[3], const double c[3],
                                   double ox, double oy, double oz, double sx, double sy,
                                   double sz) {
    double e1x = a[0] - b[0], e1y = a[1] - b[1], e1z = a[2] - b[2];
    double e2x = a[0] - c[0], e2y = a[1] - c[1], e2z = a[2] - c[2];
    double rx = a[0] - ox, ry = a[1] - oy, rz = a[2] - oz;
    double d = det3(sx, e1x, e2x, sy, e1y, e2y, sz, e1z, e2z);
    if (d == 0.0) return -1.0;
    double t = det3(rx, e1x, e2x, ry, e1y, e2y, rz, e1z, e2z) / d;
    double u = det3(sx, rx, e2x, sy, ry, e2y, sz, rz, e2z) / d;
    double w = det3(sx, e1x, rx, sy, e1y, ry, sz, e1z, rz) / d;
    if (t > EPS_T && t <= 1.0 && u >= -EPS_BARY && w >= -EPS_BARY && u + w <= 1.0 + EPS_BARY)
        return t;
    return -1.0;
}

static inline void load_tet(const om_mesh *m, int64_t e, double v[4][3]) {
    for (int j = 0; j < 4; ++j) {
        int64_t vi = m->elements[4 * e + j];
        v[j][0] = m->vertices[3 * vi + 0];
        v[j][1] = m->vertices[3 * vi + 1];
        v[j][2] = m->vertices[3 * vi + 2];
    }
}

static inline int contains_v(const double v[4][3], double px, double py, double pz,
                             double tol) {
    double l[4];
    double d = bary_core(v, px, py, pz, l);
    if (d == 0.0) return 0;
    return l[0] >= -tol && l[1] >= -tol && l[2] >= -tol && l[3] >= -tol;
}

static inline int elem_contains(const om_mesh *m, int64_t e, double px, double py,
                                double pz, double tol) {
    double v[4][3];
    load_tet(m, e, v);
    return contains_v(v, px, py, pz, tol);
}

/* kind 0 reached, 1 exit face, 2 stuck */
static inline int exit_search_core(const om_mesh *m, int64_t e, double ox, double oy,
                                   double oz, double dx, double dy, double dz, int entry,
                                   int *face_out, double *t_out) {
    double v[4][3];
    load_tet(m, e, v);
    if (contains_v(v, dx, dy, dz, EPS_BARY)) {
        *face_out = -1;
        *t_out = 1.0;
        return 0;
    }
    double sx = dx - ox, sy = dy - oy, sz = dz - oz;
    double tbest = 2.0;
    int fbest = -1;
    for (int f = 0; f < 4; ++f) {
        if (f == entry) continue;
        double t = face_hit_core(v[FV0[f]], v[FV1[f]], v[FV2[f]], ox, oy, oz, sx, sy, sz);
        if (t >= 0.0 && t < tbest - EPS_T) {
            tbest = t;
            fbest = f;
        }
    }
    if (fbest < 0) {
        *face_out = -1;
        *t_out = 0.0;
        return 2;
    }
    *face_out = fbest;
    *t_out = tbest;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* exported scalar cores (KAT tests) */

double om_bary(const double *tet12, const double *p, double *l4) {
    double v[4][3];
    memcpy(v, tet12, sizeof(v));
    return bary_core(v, p[0], p[1], p[2], l4);
}

double om_face_hit(const double *face9, const double *o, const double *s) {
    return face_hit_core(face9, face9 + 3, face9 + 6, o[0], o[1], o[2], s[0], s[1], s[2]);
}

int om_exit_search(const double *vertices, const int32_t *elements, int64_t e,
                   const double *o, const double *d, int entry, int *face, double *t) {
    om_mesh m = {vertices, elements, NULL, NULL, 0};
    return exit_search_core(&m, e, o[0], o[1], o[2], d[0], d[1], d[2], entry, face, t);
}

/* ------------------------------------------------------------------------ */
/* one fused sweep step for particle i (search.py:183-274) */

typedef struct {
    int64_t still, events, reached, boundary, recoveries, killed;
} sweep_counts;

static inline void sweep_one(const om_mesh *m, om_particles *P, int64_t i, double *slab,
                             int32_t ngroups, int score, sweep_counts *c) {
    if (P->flying[i] == 0) return;
    int64_t e = P->element[i];
    double px = P->position[3 * i], py = P->position[3 * i + 1], pz = P->position[3 * i + 2];
    double dx = P->destination[3 * i], dy = P->destination[3 * i + 1],
           dz = P->destination[3 * i + 2];
    double ox = px, oy = py, oz = pz;
    if (P->stuck[i] == 1) {
        double sx = dx - px, sy = dy - py, sz = dz - pz;
        double ln = sqrt((sx * sx + sy * sy) + sz * sz);
        if (ln > 0.0) {
            ox += NUDGE * sx / ln;
            oy += NUDGE * sy / ln;
            oz += NUDGE * sz / ln;
        }
    }
    int face;
    double t;
    int kind = exit_search_core(m, e, ox, oy, oz, dx, dy, dz, P->entry_face[i], &face, &t);
    if (kind == 2) {
        if (elem_contains(m, e, dx, dy, dz, STUCK_TOL_FACTOR * EPS_BARY)) {
            kind = 0;
            c->recoveries++;
        } else if (P->stuck[i] == 0) {
            P->stuck[i] = 1;
            c->recoveries++;
            c->still++;
            return;
        } else if (P->stuck[i] == 1) {
            int64_t hop = -1;
            for (int f = 0; f < 4; ++f) {
                int64_t nb = m->adj_elem[4 * e + f];
                if (nb >= 0 && elem_contains(m, nb, ox, oy, oz, EPS_BARY)) {
                    hop = nb;
                    break;
                }
            }
            if (hop >= 0) {
                P->element[i] = (int32_t)hop;
                P->entry_face[i] = -1;
                P->stuck[i] = 2;
                c->recoveries++;
                c->still++;
                return;
            }
            P->flying[i] = 0;
            P->alive[i] = 0;
            P->outcome[i] = OUT_STUCK_KILLED;
            c->killed++;
            return;
        } else {
            P->flying[i] = 0;
            P->alive[i] = 0;
            P->outcome[i] = OUT_STUCK_KILLED;
            c->killed++;
            return;
        }
    }
    c->events++;
    P->stuck[i] = 0;
    int64_t bin = e * ngroups + P->group[i];
    if (P->digest) {
        uint64_t code = (uint64_t)(e * 8 + face + 1);
        P->digest[i] = (P->digest[i] ^ code) * DIGEST_PRIME;
    }
    if (P->count) P->count[i] += 1;
    if (kind == 0) {
        double ax = dx - px, ay = dy - py, az = dz - pz;
        double seg = sqrt((ax * ax + ay * ay) + az * az);
        if (score) slab[bin] += P->weight[i] * seg;
        P->seg_total[i] += seg;
        P->position[3 * i] = dx;
        P->position[3 * i + 1] = dy;
        P->position[3 * i + 2] = dz;
        P->flying[i] = 0;
        P->entry_face[i] = -1;
        P->outcome[i] = OUT_REACHED;
        c->reached++;
    } else {
        double qx = ox + t * (dx - ox);
        double qy = oy + t * (dy - oy);
        double qz = oz + t * (dz - oz);
        double ax = qx - px, ay = qy - py, az = qz - pz;
        double seg = sqrt((ax * ax + ay * ay) + az * az);
        if (score) slab[bin] += P->weight[i] * seg;
        P->seg_total[i] += seg;
        P->position[3 * i] = qx;
        P->position[3 * i + 1] = qy;
        P->position[3 * i + 2] = qz;
        int64_t nb = m->adj_elem[4 * e + face];
        if (nb < 0) {
            P->flying[i] = 0;
            P->alive[i] = 0;
            P->outcome[i] = OUT_LEAKED;
            c->boundary++;
        } else {
            P->element[i] = (int32_t)nb;
            P->entry_face[i] = m->adj_face[4 * e + face];
            c->still++;
        }
    }
}

/*
 * Lockstep trace (trace_and_score).  partials: (slabs, E*G); thread t scores
 * into slab t (slabs >= threads).  Returns 0, or -1 when the sweep guard
 * (max_sweeps; <0 -> 2E+1000) is exceeded.  summary: sweeps, events, reached,
 * boundary_exits, stuck_recoveries, stuck_terminations.
 */
int om_trace(const double *vertices, const int32_t *elements, const int32_t *adj_elem,
             const int8_t *adj_face, int64_t num_elements, om_particles *P, int64_t capacity,
             double *partials, int64_t slabs, int32_t ngroups, int score, int threads,
             int64_t max_sweeps, int64_t *summary) {
    om_mesh m = {vertices, elements, adj_elem, adj_face, num_elements};
    int64_t nbins = num_elements * (int64_t)ngroups;
    int64_t limit = max_sweeps >= 0 ? max_sweeps : 2 * num_elements + 1000;
    if (threads < 1) threads = 1;
    if (slabs < threads) threads = (int)slabs;
    int64_t *active = (int64_t *)malloc(sizeof(int64_t) * (size_t)(capacity > 0 ? capacity : 1));
    int64_t mcount = 0;
    for (int64_t i = 0; i < capacity; ++i)
        if (P->flying[i] != 0) active[mcount++] = i;
    int64_t remaining = mcount, sweeps = 0;
    int64_t tot[6] = {0, 0, 0, 0, 0, 0};
    int rc = 0;
    while (remaining > 0) {
        int64_t still = 0, ev = 0, re = 0, bd = 0, rv = 0, kl = 0;
#pragma omp parallel num_threads(threads) reduction(+ : still, ev, re, bd, rv, kl)
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            double *slab = partials + (int64_t)tid * nbins;
            sweep_counts c = {0, 0, 0, 0, 0, 0};
#pragma omp for schedule(dynamic, 256)
            for (int64_t k = 0; k < mcount; ++k)
                sweep_one(&m, P, active[k], slab, ngroups, score, &c);
            still += c.still;
            ev += c.events;
            re += c.reached;
            bd += c.boundary;
            rv += c.recoveries;
            kl += c.killed;
        }
        remaining = still;
        tot[1] += ev;
        tot[2] += re;
        tot[3] += bd;
        tot[4] += rv;
        tot[5] += kl;
        sweeps++;
        if (sweeps > limit) {
            rc = -1;
            break;
        }
    }
    tot[0] = sweeps;
    memcpy(summary, tot, sizeof(tot));
    free(active);
    return rc;
}

/* _tie_break_faces (search.py:520-551), serial */
static void tie_break_faces(const om_mesh *m, om_particles *P, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        if (P->alive[i] == 0 || P->element[i] < 0) continue;
        int moved = 1;
        while (moved) {
            moved = 0;
            int64_t e = P->element[i];
            double v[4][3], l[4];
            load_tet(m, e, v);
            double px = P->position[3 * i], py = P->position[3 * i + 1],
                   pz = P->position[3 * i + 2];
            double d = bary_core(v, px, py, pz, l);
            if (d == 0.0) break;
            for (int f = 0; f < 4; ++f) {
                if (l[f] <= EPS_BARY) {
                    int64_t nb = m->adj_elem[4 * e + f];
                    if (nb >= 0 && nb < e && elem_contains(m, nb, px, py, pz, EPS_BARY)) {
                        P->element[i] = (int32_t)nb;
                        moved = 1;
                        break;
                    }
                }
            }
        }
    }
}

/*
 * initialize_locations (search.py:557-601): centroid-0 trial walk, unscored,
 * then the lost-particle reset and the tie-break.  P->destination must hold
 * the target positions for [0, count); flying[count:] must already be 0.
 * scratch_partials: at least `threads` doubles (unscored sink).
 */
int om_initialize(const double *vertices, const int32_t *elements, const int32_t *adj_elem,
                  const int8_t *adj_face, int64_t num_elements, const double *centroid0,
                  const double *bbox, om_particles *P, int64_t count, int64_t capacity,
                  int threads, int64_t *summary) {
    om_mesh m = {vertices, elements, adj_elem, adj_face, num_elements};
    for (int64_t i = count; i < capacity; ++i) P->flying[i] = 0;
    for (int64_t i = 0; i < count; ++i) {
        const double *p = P->destination + 3 * i;
        int inside = 1;
        for (int a = 0; a < 3; ++a)
            if (!(p[a] >= bbox[a] && p[a] <= bbox[3 + a])) inside = 0;
        P->position[3 * i] = centroid0[0];
        P->position[3 * i + 1] = centroid0[1];
        P->position[3 * i + 2] = centroid0[2];
        P->element[i] = inside ? 0 : -1;
        P->flying[i] = (int8_t)inside;
        P->alive[i] = (int8_t)inside;
        P->entry_face[i] = -1;
        P->stuck[i] = 0;
        P->outcome[i] = OUT_NONE;
        P->seg_total[i] = 0.0;
    }
    double *sink = (double *)calloc((size_t)(threads > 0 ? threads : 1), sizeof(double));
    om_particles Q = *P;
    Q.digest = NULL;
    Q.count = NULL;
    /* unscored: the sink grid is 1x1; score=0 never touches it */
    int rc = om_trace(vertices, elements, adj_elem, adj_face, 1, &Q, capacity, sink,
                      threads > 0 ? threads : 1, 1, 0, threads, 2 * num_elements + 1000,
                      summary);
    free(sink);
    (void)m;
    for (int64_t i = 0; i < count; ++i)
        if (P->outcome[i] == OUT_LEAKED || P->outcome[i] == OUT_STUCK_KILLED) P->element[i] = -1;
    tie_break_faces(&m, P, count);
    return rc;
}

/* lowest-id element containing each point (exhaustive; small meshes only) --
 * the semantics of pkg/tests/oracles.py:36-57 with the reference's own bary
 * arithmetic and EPS_BARY. */
void om_locate_exhaustive(const double *vertices, const int32_t *elements,
                          int64_t num_elements, const double *pts, int64_t n, int32_t *out,
                          int threads) {
    om_mesh m = {vertices, elements, NULL, NULL, num_elements};
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
        int32_t found = -1;
        for (int64_t e = 0; e < num_elements; ++e)
            if (elem_contains(&m, e, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], EPS_BARY)) {
                found = (int32_t)e;
                break;
            }
        out[i] = found;
    }
}

/* _finalize (tally.py:83-95) */
void om_finalize(double *partials, int64_t slabs, int64_t nbins, double source_weight,
                 double *sum, double *sum_sq) {
    for (int64_t b = 0; b < nbins; ++b) {
        double acc = 0.0;
        for (int64_t s = 0; s < slabs; ++s) {
            acc += partials[s * nbins + b];
            partials[s * nbins + b] = 0.0;
        }
        double x = acc / source_weight;
        sum[b] += x;
        sum_sq[b] += x * x;
    }
}

int om_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ======================================================================== */
/* Transport driver: philox4x64-10 (rng.py:16-64) and the
 * event loop of transport.run (transport.py:445-549) with _source (154-181),
 * _trial_setup (184-201), _rearm (204-210), _flight (213-226) and _collide
 * (229-275).  Serial (threads = 1) to reproduce the reference's summation
 * order exactly.  log/cos/sin come from the C library, as numba's do. */

static const uint64_t PH_M0 = 0xD2E7470EE14C6C93ULL, PH_M1 = 0xCA5A826395121157ULL;
static const uint64_t PH_W0 = 0x9E3779B97F4A7C15ULL, PH_W1 = 0xBB67AE8584CAA73BULL;
static const uint64_t PH_KEY1 = 0xD1B54A32D192ED03ULL;

void om_philox(const uint64_t *ctr, const uint64_t *key, uint64_t *out) {
    uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        __uint128_t p0 = (__uint128_t)PH_M0 * c0, p1 = (__uint128_t)PH_M1 * c2;
        uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
        uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += PH_W0;
        k1 += PH_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void om_uniform_block(uint64_t seed, uint64_t batch, uint64_t particle, uint64_t block,
                      double *u) {
    uint64_t ctr[4] = {block, particle, batch, 0}, key[2] = {seed, PH_KEY1}, w[4];
    om_philox(ctr, key, w);
    for (int j = 0; j < 4; ++j) u[j] = ((double)(w[j] >> 11) + 1.0) * (1.0 / 9007199254740992.0);
}

typedef struct {
    int64_t ng;
    const double *sigma_t;      /* (G) */
    const double *scatter_prob; /* (G)  = rowsum(sigma_s)/sigma_t  (XSData) */
    const double *group_cdf;    /* (G,G) */
} om_xs;

/* totals: source_w, leaked_w, absorbed_w, stuck_w, collisions, events, sweeps, track_total */
int om_transport_run(const double *vertices, const int32_t *elements, const int32_t *adj_elem,
                     const int8_t *adj_face, int64_t ne, const double *centroid0,
                     int64_t ng, const double *sigma_t, const double *scatter_prob,
                     const double *group_cdf, int64_t n, int64_t num_batches, uint64_t seed,
                     const double *box, int fixed_dir, const double *fd, double *track_partials,
                     double *track_sum, double *track_sum_sq, double *col_partials,
                     double *col_sum, double *col_sum_sq, double *totals, om_particles *P,
                     double *direction, int32_t *group_out, uint64_t *rng_block) {
    om_mesh m = {vertices, elements, adj_elem, adj_face, ne};
    (void)m;
    double *dest = (double *)P->destination; /* the caller gives a writable buffer */
    double *weight = (double *)P->weight;
    int32_t *group = (int32_t *)P->group;
    int64_t nb = ne * ng;
    double source_w = 0, leaked_w = 0, absorbed_w = 0, stuck_w = 0, track_total = 0;
    int64_t collisions = 0, events = 0, sweeps = 0;
    int64_t *active = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t summ[6];
    double sink = 0.0;
    for (int64_t b = 0; b < num_batches; ++b) {
        /* _source */
        for (int64_t i = 0; i < n; ++i) {
            double u[4];
            om_uniform_block(seed, (uint64_t)b, (uint64_t)i, 0, u);
            dest[3 * i] = box[0] + (box[3] - box[0]) * u[0];
            dest[3 * i + 1] = box[1] + (box[4] - box[1]) * u[1];
            dest[3 * i + 2] = box[2] + (box[5] - box[2]) * u[2];
            if (fixed_dir) {
                direction[3 * i] = fd[0];
                direction[3 * i + 1] = fd[1];
                direction[3 * i + 2] = fd[2];
            } else {
                double v[4];
                om_uniform_block(seed, (uint64_t)b, (uint64_t)i, 1, v);
                double mu = 2.0 * v[0] - 1.0;
                double phi = (2.0 * 3.141592653589793) * v[1];
                double t = 1.0 - mu * mu;
                double s = sqrt(t > 0.0 ? t : 0.0);
                direction[3 * i] = s * cos(phi);
                direction[3 * i + 1] = s * sin(phi);
                direction[3 * i + 2] = mu;
            }
            weight[i] = 1.0;
            group[i] = 0;
            P->alive[i] = 1;
            P->flying[i] = 0;
            rng_block[i] = 2;
            P->outcome[i] = OUT_NONE;
        }
        /* _trial_setup + unscored walk + tie-break (_localize_adjacency) */
        for (int64_t i = 0; i < n; ++i) {
            P->position[3 * i] = centroid0[0];
            P->position[3 * i + 1] = centroid0[1];
            P->position[3 * i + 2] = centroid0[2];
            P->element[i] = 0;
            P->flying[i] = P->alive[i];
            P->entry_face[i] = -1;
            P->stuck[i] = 0;
            P->seg_total[i] = 0.0;
        }
        om_particles Q = *P;
        Q.digest = NULL;
        Q.count = NULL;
        if (om_trace(vertices, elements, adj_elem, adj_face, ne, &Q, n, &sink, 1, 1, 0, 1,
                     2 * ne + 1000, summ) != 0)
            return -1;
        tie_break_faces(&m, P, n);
        /* _rearm */
        for (int64_t i = 0; i < n; ++i) {
            P->flying[i] = P->alive[i];
            P->entry_face[i] = -1;
            P->outcome[i] = OUT_NONE;
            P->seg_total[i] = 0.0;
        }
        /* batch source weight: weight[:n][alive].sum() (all weights are 1.0) */
        double bsw = 0.0;
        for (int64_t i = 0; i < n; ++i)
            if (P->alive[i]) bsw += weight[i];
        source_w += bsw;
        for (;;) {
            int64_t mcount = 0;
            for (int64_t i = 0; i < n; ++i)
                if (P->flying[i]) active[mcount++] = i;
            if (mcount == 0) break;
            /* _flight */
            for (int64_t k = 0; k < mcount; ++k) {
                int64_t i = active[k];
                double u[4];
                om_uniform_block(seed, (uint64_t)b, (uint64_t)i, rng_block[i], u);
                rng_block[i] += 1;
                double lc = -log(u[0]) / sigma_t[group[i]];
                dest[3 * i] = P->position[3 * i] + lc * direction[3 * i];
                dest[3 * i + 1] = P->position[3 * i + 1] + lc * direction[3 * i + 1];
                dest[3 * i + 2] = P->position[3 * i + 2] + lc * direction[3 * i + 2];
                P->outcome[i] = OUT_NONE;
            }
            if (om_trace(vertices, elements, adj_elem, adj_face, ne, &Q, n, track_partials, 1,
                         (int32_t)ng, 1, 1, 2 * ne + 1000, summ) != 0)
                return -1;
            events += summ[1];
            sweeps += summ[0];
            /* _collide */
            for (int64_t k = 0; k < mcount; ++k) {
                int64_t i = active[k];
                int8_t oc = P->outcome[i];
                if (oc == OUT_REACHED) {
                    int32_t g = group[i];
                    double w = weight[i];
                    int64_t e = P->element[i];
                    col_partials[e * ng + g] += w / sigma_t[g];
                    collisions += 1;
                    double u[4];
                    om_uniform_block(seed, (uint64_t)b, (uint64_t)i, rng_block[i], u);
                    rng_block[i] += 1;
                    if (u[0] <= scatter_prob[g]) {
                        int32_t gp = 0;
                        for (int64_t j = 0; j < ng; ++j) {
                            gp = (int32_t)j;
                            if (u[1] <= group_cdf[g * ng + j]) break;
                        }
                        double mu = 2.0 * u[2] - 1.0;
                        double phi = (2.0 * 3.141592653589793) * u[3];
                        double t = 1.0 - mu * mu;
                        double s = sqrt(t > 0.0 ? t : 0.0);
                        direction[3 * i] = s * cos(phi);
                        direction[3 * i + 1] = s * sin(phi);
                        direction[3 * i + 2] = mu;
                        group[i] = gp;
                        P->flying[i] = 1;
                    } else {
                        P->alive[i] = 0;
                        P->flying[i] = 0;
                        P->outcome[i] = 5; /* OUTCOME_ABSORBED */
                        absorbed_w += w;
                    }
                } else if (oc == OUT_LEAKED) {
                    leaked_w += weight[i];
                } else if (oc == OUT_STUCK_KILLED) {
                    stuck_w += weight[i];
                }
            }
        }
        double ts = 0.0;
        for (int64_t i = 0; i < n; ++i) ts += P->seg_total[i];
        track_total += ts;
        om_finalize(track_partials, 1, nb, bsw, track_sum, track_sum_sq);
        om_finalize(col_partials, 1, nb, bsw, col_sum, col_sum_sq);
    }
    for (int64_t i = 0; i < n; ++i) group_out[i] = group[i];
    free(active);
    totals[0] = source_w;
    totals[1] = leaked_w;
    totals[2] = absorbed_w;
    totals[3] = stuck_w;
    totals[4] = (double)collisions;
    totals[5] = (double)events;
    totals[6] = (double)sweeps;
    totals[7] = track_total;
    return 0;
}
