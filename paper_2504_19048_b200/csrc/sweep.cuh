// sweep.cuh -- Listing-1 callback path, load_step, digests, flux.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

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
