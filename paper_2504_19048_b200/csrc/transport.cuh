// transport.cuh -- device transport: philox, source, histories.
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

// ---------------------------------------------------------------------------
// Transport: the reference's event loop (transport.run,
// transport.py:445-549) alternates flight / walk / collide over all flying
// particles.  Particles never interact and every random draw is keyed by
// (seed, batch, particle, block) (rng.py:58-64), so each particle's history
// is the same whether it is advanced event by event or to completion: one
// lane runs a whole history (flight -> walk with track-length scoring ->
// collision estimator + scatter/absorb -> ...) in a persistent kernel.

constexpr uint64_t PH_M0 = 0xD2E7470EE14C6C93ull, PH_M1 = 0xCA5A826395121157ull;
constexpr uint64_t PH_W0 = 0x9E3779B97F4A7C15ull, PH_W1 = 0xBB67AE8584CAA73Bull;
constexpr uint64_t PH_KEY1 = 0xD1B54A32D192ED03ull;
constexpr double TWO_PI = 2.0 * 3.141592653589793;

// philox4x64-10 block (rng.py:38-49) -> four uniforms in (0, 1] (rng.py:52-64)
__device__ __forceinline__ void uniform_block(uint64_t seed, uint64_t batch, uint64_t particle,
                                              uint64_t block, double u[4]) {
    uint64_t c0 = block, c1 = particle, c2 = batch, c3 = 0, k0 = seed, k1 = PH_KEY1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t hi0 = __umul64hi(PH_M0, c0), lo0 = PH_M0 * c0;
        const uint64_t hi1 = __umul64hi(PH_M1, c2), lo1 = PH_M1 * c2;
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += PH_W0;
        k1 += PH_W1;
    }
    const double s = 1.0 / 9007199254740992.0;
    u[0] = __dmul_rn(__dadd_rn((double)(c0 >> 11), 1.0), s);
    u[1] = __dmul_rn(__dadd_rn((double)(c1 >> 11), 1.0), s);
    u[2] = __dmul_rn(__dadd_rn((double)(c2 >> 11), 1.0), s);
    u[3] = __dmul_rn(__dadd_rn((double)(c3 >> 11), 1.0), s);
}

__global__ void philox_kat_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                  double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uniform_block(keys[4 * i], keys[4 * i + 1], keys[4 * i + 2], keys[4 * i + 3], out + 4 * i);
}

// The reference's np.log / np.cos / np.sin are the host libm's: with its
// tables available (BT_GLIBC_MATH, glibc_math.cuh) the device evaluates the
// same operation sequences and every history is the reference's bit for bit;
// otherwise CUDA's functions (last-bit differences: statistical parity only).
__device__ __forceinline__ double tr_log(double x) {
#if BT_GLIBC_MATH
    return gm_log(x);
#else
    return log(x);
#endif
}
__device__ __forceinline__ void tr_sincos(double phi, double* sp, double* cp) {
#if BT_GLIBC_MATH
    gm_sincos_simt(phi, sp, cp);
#else
    sincos(phi, sp, cp);
#endif
}

// isotropic direction from two uniforms (transport.py:172-178, 255-261)
__device__ __forceinline__ void iso_dir(double ua, double ub, double& x, double& y, double& z) {
    const double mu = __dsub_rn(__dmul_rn(2.0, ua), 1.0);
    const double phi = __dmul_rn(TWO_PI, ub);
    const double t = __dsub_rn(1.0, __dmul_rn(mu, mu));
    const double s = __dsqrt_rn(t > 0.0 ? t : 0.0);
    double sp, cp;
    tr_sincos(phi, &sp, &cp);
    x = __dmul_rn(s, cp);
    y = __dmul_rn(s, sp);
    z = mu;
}

struct XSDev {
    const double* sigma_t;      // (G)
    const double* scatter_prob; // (G)
    const double* group_cdf;    // (G,G)
    int32_t ng;
};

struct TransportArgs {
    WalkArgs w;                 // mesh, particle state, track tally (w.tally)
    XSDev xs;
    double* col_tally;          // collision estimator (E*G)
    double* dir;                // (N,3)
    uint32_t* rng_block;        // (N)
    int32_t* group_rw;          // (N) groups (written)
    double* weight_rw;          // (N)
    const double* src;          // (n,3) source positions (located)
    unsigned* round_max;        // per-round max walk steps (sweeps), MAX_ROUNDS_TRACKED
    unsigned long long* tcount; // [0] collisions [1] rounds overflow [2] lost
    double* wsum;               // [0] leaked [1] absorbed [2] stuck [3] track length
    unsigned long long* queue;
    uint64_t seed, batch;
    int64_t n;
    int64_t max_rounds;
};

constexpr int MAX_ROUNDS_TRACKED = 1 << 20;

// per-batch source sampling (transport.py:154-181), blocks 0 and 1
__global__ void transport_source_kernel(TransportArgs a, double box0, double box1, double box2,
                                        double box3, double box4, double box5, int fixed,
                                        double fdx, double fdy, double fdz,
                                        double* __restrict__ stage) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    double u[4];
    uniform_block(a.seed, a.batch, i, 0, u);
    stage[3 * i] = __dadd_rn(box0, __dmul_rn(__dsub_rn(box3, box0), u[0]));
    stage[3 * i + 1] = __dadd_rn(box1, __dmul_rn(__dsub_rn(box4, box1), u[1]));
    stage[3 * i + 2] = __dadd_rn(box2, __dmul_rn(__dsub_rn(box5, box2), u[2]));
    double dx = fdx, dy = fdy, dz = fdz;
    if (!fixed) {
        double v[4];
        uniform_block(a.seed, a.batch, i, 1, v);
        iso_dir(v[0], v[1], dx, dy, dz);
    }
    a.dir[3 * i] = dx;
    a.dir[3 * i + 1] = dy;
    a.dir[3 * i + 2] = dz;
    a.weight_rw[i] = 1.0;
    a.group_rw[i] = 0;
    a.rng_block[i] = 2;
}

// one history per lane, persistent; refill from a global counter
template <int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) transport_kernel(const TransportArgs t) {
    static_assert(THREADS <= MAX_CTA_THREADS, "one shared lane slot per thread");
    constexpr unsigned FULL = 0xffffffffu;
    const WalkArgs& a = t.w;
    const int lane = threadIdx.x & 31;
    __shared__ unsigned shc[SC_N];
    VSLOTS_DECL(THREADS)
    counters_init(shc);
    const DigestSlot DS{nullptr, nullptr};
    Lane L;
    L.busy = false;
    VSLOTS_INIT(L);
    Counters C;
    C.sh = shc;
    Pending P;
    P.init(a);
    // direction and the per-lane totals, touched once per flight: shared
    // slots keep them out of the walk step's registers
    __shared__ double s_tr[6][THREADS];
    __shared__ unsigned s_col[THREADS];
    double& ux = s_tr[0][threadIdx.x];
    double& uy = s_tr[1][threadIdx.x];
    double& uz = s_tr[2][threadIdx.x];
    double& leaked = s_tr[3][threadIdx.x];
    double& absorbed = s_tr[4][threadIdx.x];
    double& stuck_w = s_tr[5][threadIdx.x];
    unsigned& collisions = s_col[threadIdx.x];
    ux = uy = uz = 0.0;
    leaked = absorbed = stuck_w = 0.0;
    collisions = 0;
    uint32_t rb = 0;
    int rounds = 0;
    bool drained = false;
    bool need_flight = false;
    while (true) {
        if (!drained) {
            const unsigned idle = __ballot_sync(FULL, !L.busy);
            if (idle) {
                const unsigned nidle = __popc(idle);
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(t.queue, (unsigned long long)nidle);
                base = __shfl_sync(FULL, base, 0);
                if (base + nidle >= (unsigned long long)t.n) drained = true;
                if (!L.busy) {
                    const unsigned long long q = base + __popc(idle & lanemask_lt());
                    if (q < (unsigned long long)t.n && a.alive[q]) {
                        const int64_t i = (int64_t)q;
                        L.set_idx(i);
                        L.e = a.element[i];
                        L.px = a.pos[3 * i];
                        L.py = a.pos[3 * i + 1];
                        L.pz = a.pos[3 * i + 2];
                        L.seg() = 0.0;
                        L.w() = t.weight_rw[i];
                        L.g() = t.group_rw[i];
                        ux = t.dir[3 * i];
                        uy = t.dir[3 * i + 1];
                        uz = t.dir[3 * i + 2];
                        rb = t.rng_block[i];
                        L.entry = -1;
                        L.st = 0;
                        vslots_fill(a, L, L.e, elem_vids(a, L.e));  // a new history
                        rounds = 0;
                        need_flight = true;
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
            if (need_flight) {  // _flight (transport.py:213-226)
                double u[4];
                uniform_block(t.seed, t.batch, (uint64_t)L.idx(), rb, u);
                ++rb;
                const double lc = __ddiv_rn(-tr_log(u[0]), t.xs.sigma_t[L.g()]);
                L.dx() = __dadd_rn(L.px, __dmul_rn(lc, ux));
                L.dy() = __dadd_rn(L.py, __dmul_rn(lc, uy));
                L.dz() = __dadd_rn(L.pz, __dmul_rn(lc, uz));
                L.iters = 0;
                L.outcome() = OUT_NONE;
                L.alive() = 1;
                ++rounds;
                need_flight = false;
            }
            if (walk_step<false>(a, L, C, P, DS)) {
                sweep_guard_hit(a, L, C);
                // flight over: its walk took L.iters sweeps in round `rounds`
                if (rounds <= MAX_ROUNDS_TRACKED) atomicMax(t.round_max + rounds - 1, (unsigned)L.iters);
                bool stop = true;
                if (L.outcome() == OUT_REACHED) {  // _collide (transport.py:229-275)
                    const int g = L.g();
                    const double st_g = t.xs.sigma_t[g];
                    atomicAdd(t.col_tally + (int64_t)L.e * t.xs.ng + g, __ddiv_rn(L.w(), st_g));
                    ++collisions;
                    double u[4];
                    uniform_block(t.seed, t.batch, (uint64_t)L.idx(), rb, u);
                    ++rb;
                    if (u[0] <= t.xs.scatter_prob[g]) {
                        int gp = 0;
                        for (int j = 0; j < t.xs.ng; ++j) {
                            gp = j;
                            if (u[1] <= t.xs.group_cdf[g * t.xs.ng + j]) break;
                        }
                        iso_dir(u[2], u[3], ux, uy, uz);
                        L.g() = gp;
                        stop = false;
                        need_flight = true;
                        if (rounds >= t.max_rounds) {  // _MAX_ROUNDS guard (transport.py:531-533)
                            atomicOr(C.sh + SC_ERR, 1u);
                            stop = true;
                        }
                    } else {
                        L.alive() = 0;
                        L.outcome() = 5;  // OUTCOME_ABSORBED
                        absorbed += L.w();
                    }
                } else if (L.outcome() == OUT_LEAKED) {
                    leaked += L.w();
                } else if (L.outcome() == OUT_STUCK_KILLED) {
                    stuck_w += L.w();
                }
                if (stop) {
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
                    t.dir[3 * i] = ux;
                    t.dir[3 * i + 1] = uy;
                    t.dir[3 * i + 2] = uz;
                    t.rng_block[i] = rb;
                    t.group_rw[i] = L.g();
                    L.busy = false;
                }
            }
        }
        flush_pending(a, P, !L.busy);
    }
    // reduce the per-lane totals (tally sums are order-free up to rounding)
    double lk = leaked, ab = absorbed, sw = stuck_w;
    for (int o = 16; o > 0; o >>= 1) {
        lk += __shfl_xor_sync(FULL, lk, o);
        ab += __shfl_xor_sync(FULL, ab, o);
        sw += __shfl_xor_sync(FULL, sw, o);
    }
    const unsigned cl = __reduce_add_sync(FULL, collisions);
    if (lane == 0) {
        if (lk != 0.0) atomicAdd(t.wsum + 0, lk);
        if (ab != 0.0) atomicAdd(t.wsum + 1, ab);
        if (sw != 0.0) atomicAdd(t.wsum + 2, sw);
        if (cl) atomicAdd(t.tcount + 0, (unsigned long long)cl);
    }
    flush_counters(a, C);
}

__global__ void sum_rounds_kernel(const unsigned* __restrict__ round_max, int64_t n,
                                  unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        s += round_max[r];
    s = __reduce_add_sync(0xffffffffu, (unsigned)s);  // per-warp (< 2^32 per warp chunk)
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

__global__ void seg_sum_kernel(const double* __restrict__ seg, const int8_t* __restrict__ alive0,
                               int64_t n, double* __restrict__ out) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += seg[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(out, s);
}

__global__ void count_alive_kernel(const int8_t* __restrict__ alive, int64_t n,
                                   unsigned long long* __restrict__ out) {
    unsigned c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        c += alive[i] != 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}
