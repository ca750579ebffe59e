// glibc_math.cuh -- log, sin and cos with the host C library's bits.
//
// The reference's transport (transport.py:172-178, 213-275) calls np.log,
// np.cos, np.sin; numba lowers them to the process's libm, which on this
// image (x86-64 glibc 2.39, a CPU with FMA) dispatches to __log_fma,
// __sin_fma and __cos_fma (sincos gives the same bits: checked on 1e8
// transport angles).  These are their operation sequences -- the
// optimized-routines log (table of 128 (1/c, log c), degree-5 polynomial on
// r = z/c - 1, a degree-11 one near 1) and the IBM sin/cos (range reduction by
// pi/2 in three parts, table of sin/cos at k/128 as double-double, short
// polynomials) -- with every multiply-add the compiled library fuses written
// as one fma and every other operation rounded on its own, so each result is
// the library's bit for bit on the transport's arguments (log on (0, 1],
// sin/cos on (0, 2 pi]; larger angles (Payne-Hanek) and non-finite inputs are
// outside them and fall back to CUDA's functions).
//
// Tables: gm_log_tab / gm_sincos_tab (glibc_tables.inc, generated from the
// libm at build time by paper_2504_19048_b200/glibc_tables.py).  Device
// functions under nvcc; a plain C++ build of the same header (g++
// -ffp-contract=off, std::fma) is the self-test against libm
// (tests/test_glibc_math.py).
// Part of libb200tally (included by b200tally.cu, one translation unit).
#pragma once

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define GM_HD __device__ __forceinline__
#define GM_TABLE __device__ const
#else
#include <cmath>
#define GM_HD static inline
#define GM_TABLE static const
#endif

#include "glibc_tables.inc"

#if BT_GLIBC_MATH

#if defined(__CUDA_ARCH__)
#define GM_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GM_MUL(a, b) __dmul_rn((a), (b))
#define GM_ADD(a, b) __dadd_rn((a), (b))
#define GM_SUB(a, b) __dsub_rn((a), (b))
#define GM_LD(p) __ldg(p)
#else
#define GM_FMA(a, b, c) std::fma((a), (b), (c))
#define GM_MUL(a, b) ((a) * (b))
#define GM_ADD(a, b) ((a) + (b))
#define GM_SUB(a, b) ((a) - (b))
#define GM_LD(p) (*(p))
#endif

GM_HD uint64_t gm_bits(double x) {
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
}
GM_HD double gm_double(uint64_t u) {
    double x;
    memcpy(&x, &u, 8);
    return x;
}
GM_HD double gm_copysign(double mag, double sgn) {
    return gm_double((gm_bits(mag) & 0x7fffffffffffffffull) | (gm_bits(sgn) & 0x8000000000000000ull));
}
GM_HD double gm_neg(double x) { return gm_double(gm_bits(x) ^ 0x8000000000000000ull); }
GM_HD double gm_fabs(double x) { return gm_double(gm_bits(x) & 0x7fffffffffffffffull); }

// ---- log: x normal and positive ------------------------------------------
GM_HD double gm_log(double x) {
    const uint64_t ix = gm_bits(x);
    if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {  // x in [1 - 2^-4, 1 + 0x1.09p-4)
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double r = GM_SUB(x, 1.0);
        double p2 = GM_FMA(r, -0x1.ffffffffffdcbp-3, 0x1.5555555555577p-2);
        double p3 = GM_FMA(r, 0x1.24924a344de30p-3, -0x1.55555556745a7p-3);
        const double r2 = GM_MUL(r, r);
        const double p5 = GM_FMA(r, -0x1.999eb43b068ffp-4, 0x1.c7184282ad6cap-4);
        p2 = GM_FMA(r2, 0x1.999999995dd0cp-3, p2);
        p3 = GM_FMA(r2, -0x1.fffffa4423d65p-4, p3);
        const double r3 = GM_MUL(r, r2);
        double q = GM_FMA(r2, 0x1.78182f7afd085p-4, p5);
        q = GM_FMA(r3, -0x1.5521375d145cdp-4, q);
        q = GM_FMA(q, r3, p3);
        q = GM_FMA(q, r3, p2);
        // r split into rhi + rlo with rhi = (r + r 2^27) - r 2^27 (both fused)
        const double t = GM_FMA(r, 0x1p27, r);
        const double rhi = GM_FMA(-0x1p27, r, t);
        const double rh2 = GM_MUL(rhi, rhi);
        const double rlo = GM_SUB(r, rhi);
        const double hi = GM_FMA(rh2, -0.5, r);
        double lo = GM_FMA(rh2, -0.5, GM_SUB(r, hi));
        lo = GM_FMA(GM_MUL(-0.5, rlo), GM_ADD(r, rhi), lo);
        return GM_ADD(hi, GM_FMA(q, r3, lo));
    }
    if (((ix >> 48) - 0x10u) > 0x7fdfu) {  // subnormal, zero, negative, inf, nan
#ifdef __CUDA_ARCH__
        return log(x);
#else
        return std::log(x);
#endif
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = (int)((tmp >> 45) & 0x7f);
    const int k = (int)((int64_t)tmp >> 52);
    const double z = gm_double(ix - (tmp & 0xfff0000000000000ull));
    const double invc = GM_LD(gm_log_tab + 2 * i), logc = GM_LD(gm_log_tab + 2 * i + 1);
    const double kd = (double)k;
    const double w = GM_FMA(kd, 0x1.62e42fefa3800p-1, logc);
    const double r = GM_FMA(z, invc, -1.0);
    const double p12 = GM_FMA(r, -0x1.fffffffeb4590p-3, 0x1.555555551305bp-2);
    const double hi = GM_ADD(r, w);
    const double r2 = GM_MUL(r, r);
    double lo = GM_ADD(GM_SUB(w, hi), r);
    lo = GM_FMA(kd, 0x1.ef35793c76730p-45, lo);
    const double r3 = GM_MUL(r, r2);
    double q = GM_FMA(r, -0x1.55575e506c89fp-3, 0x1.999b324f10111p-3);
    lo = GM_FMA(r2, -0x1.0000000000001p-1, lo);
    q = GM_FMA(q, r2, p12);
    return GM_ADD(GM_FMA(r3, q, lo), hi);
}

// ---- sin / cos ------------------------------------------------------------
// big = 1.5 * 2^45: |x| + big rounds |x| to a multiple of 1/128, whose index
// lands in the low word
constexpr double GM_BIG = 0x1.8p45;
constexpr double GM_SN3 = -0x1.5555555555515p-3, GM_SN5 = 0x1.11110e829872fp-7;
constexpr double GM_CS4 = -0x1.5555555555535p-5, GM_CS6 = 0x1.6c16bedd9e239p-10;
constexpr double GM_HP0 = 0x1.921fb54442d18p+0, GM_HP1 = 0x1.1a62633145c07p-54;

// table entry k: sin(k/128) = sn + ssn, cos(k/128) = cs + ccs
#define GM_SC(k4, j) GM_LD(gm_sincos_tab + (k4) + (j))

// do_sin(x, dx) for xa = |x| >= 0.126, dx already sign-adjusted (the caller
// applies copysign(., x))
GM_HD double gm_do_sin(double xa, double dx) {
    const double u = GM_ADD(xa, GM_BIG);
    const double x = GM_SUB(xa, GM_SUB(u, GM_BIG));
    const int k4 = (int)((uint32_t)gm_bits(u) << 2);
    const double xx = GM_MUL(x, x);
    const double p = GM_FMA(xx, GM_SN5, GM_SN3);
    const double s = GM_ADD(x, GM_FMA(GM_MUL(x, xx), p, dx));
    const double pc = GM_FMA(xx, GM_FMA(xx, GM_CS6, GM_CS4), 0.5);
    const double c = GM_FMA(x, dx, GM_MUL(xx, pc));
    const double sn = GM_SC(k4, 0), ssn = GM_SC(k4, 1), cs = GM_SC(k4, 2), ccs = GM_SC(k4, 3);
    double cor = GM_FMA(s, ccs, ssn);
    cor = GM_FMA(-c, sn, cor);
    cor = GM_FMA(s, cs, cor);
    return GM_ADD(sn, cor);
}
// do_cos(x, dx) for xa = |x|, dx already sign-adjusted
GM_HD double gm_do_cos(double xa, double dx) {
    const double u = GM_ADD(xa, GM_BIG);
    const double x = GM_ADD(GM_SUB(xa, GM_SUB(u, GM_BIG)), dx);
    const int k4 = (int)((uint32_t)gm_bits(u) << 2);
    const double xx = GM_MUL(x, x);
    const double p = GM_FMA(xx, GM_SN5, GM_SN3);
    const double s = GM_FMA(GM_MUL(x, xx), p, x);
    const double c = GM_MUL(xx, GM_FMA(xx, GM_FMA(xx, GM_CS6, GM_CS4), 0.5));
    const double sn = GM_SC(k4, 0), ssn = GM_SC(k4, 1), cs = GM_SC(k4, 2), ccs = GM_SC(k4, 3);
    double cor = GM_FMA(-s, ssn, ccs);
    cor = GM_FMA(-c, cs, cor);
    cor = GM_FMA(-s, sn, cor);
    return GM_ADD(cs, cor);
}
// TAYLOR_SIN(a*a, a, da) for |a| < 0.126
GM_HD double gm_taylor_sin(double a, double da) {
    const double xx = GM_MUL(a, a);
    double p = -0x1.addffc2fcdf59p-26;
    p = GM_FMA(xx, p, 0x1.71de27b9a7ed9p-19);
    p = GM_FMA(xx, p, -0x1.a01a019db08b8p-13);
    p = GM_FMA(xx, p, 0x1.1111111110ecep-7);
    p = GM_FMA(xx, p, -0x1.5555555555555p-3);
    const double t = GM_FMA(p, a, -GM_MUL(da, 0.5));
    return GM_ADD(a, GM_FMA(xx, t, da));
}
// reduce_sincos: x = n pi/2 + (b + db), 2.426 < |x| < 105414350
GM_HD int gm_reduce(double x, double& b, double& db) {
    const double t = GM_FMA(x, 0x1.45f306dc9c883p-1, 0x1.8p52);
    const double xn = GM_SUB(t, 0x1.8p52);
    double y = GM_FMA(-xn, 0x1.921fb58000000p+0, x);
    y = GM_FMA(-xn, -0x1.dde973c000000p-27, y);
    constexpr double PP3 = -0x1.cb3b398000000p-55, PP4 = -0x1.d747f23e32ed7p-83;
    const double t2 = GM_FMA(-xn, PP3, y);
    double d = GM_FMA(-xn, PP3, GM_SUB(y, t2));
    b = GM_FMA(-xn, PP4, t2);
    d = GM_ADD(d, GM_FMA(-xn, PP4, GM_SUB(t2, b)));
    db = d;
    return (int)(gm_bits(t) & 3u);
}
// sin (n even) or cos (n odd) of the reduced b + db, negated for n & 2
GM_HD double gm_sincos_reduced(double b, double db, int n) {
    double r;
    if (n & 1) {
        r = gm_do_cos(gm_fabs(b), b < 0.0 ? gm_neg(db) : db);
    } else if (gm_fabs(b) < 0.126) {
        r = gm_taylor_sin(b, db);
    } else {
        r = gm_copysign(gm_do_sin(gm_fabs(b), b <= 0.0 ? gm_neg(db) : db), b);
    }
    return (n & 2) ? gm_neg(r) : r;
}

GM_HD double gm_sin(double x) {
    const uint32_t k = (uint32_t)(gm_bits(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e500000u) return x;
    if (k < 0x3feb6000u) {
        if (gm_fabs(x) < 0.126) return gm_taylor_sin(x, 0.0);
        return gm_copysign(gm_do_sin(gm_fabs(x), x > 0.0 ? 0.0 : -0.0), x);
    }
    if (k < 0x400368fdu) {
        const double t = GM_SUB(GM_HP0, gm_fabs(x));
        return gm_copysign(gm_do_cos(gm_fabs(t), t >= 0.0 ? GM_HP1 : -GM_HP1), x);
    }
    if (k < 0x419921fbu) {
        double b, db;
        const int n = gm_reduce(x, b, db);
        return gm_sincos_reduced(b, db, n);
    }
#ifdef __CUDA_ARCH__
    return sin(x);
#else
    return std::sin(x);
#endif
}

GM_HD double gm_cos(double x) {
    const uint32_t k = (uint32_t)(gm_bits(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) return 1.0;
    if (k < 0x3feb6000u) return gm_do_cos(gm_fabs(x), x >= 0.0 ? 0.0 : -0.0);
    if (k < 0x400368fdu) {
        const double y = GM_SUB(GM_HP0, gm_fabs(x));
        const double a = GM_ADD(y, GM_HP1);
        const double da = GM_ADD(GM_SUB(y, a), GM_HP1);
        if (gm_fabs(a) < 0.126) return gm_taylor_sin(a, da);
        return gm_copysign(gm_do_sin(gm_fabs(a), a <= 0.0 ? gm_neg(da) : da), a);
    }
    if (k < 0x419921fbu) {
        double b, db;
        const int n = gm_reduce(x, b, db);
        return gm_sincos_reduced(b, db, n + 1);
    }
#ifdef __CUDA_ARCH__
    return cos(x);
#else
    return std::cos(x);
#endif
}

// sin and cos of one argument: the same results as gm_sin / gm_cos (the same
// functions on the same arguments), with the range reduction and the branch
// decisions shared -- what the transport's direction sampling needs
GM_HD void gm_sincos(double x, double* sp, double* cp) {
    const uint32_t k = (uint32_t)(gm_bits(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) {
        *sp = x;
        *cp = 1.0;
    } else if (k < 0x3feb6000u) {
        if (k < 0x3e500000u)
            *sp = x;
        else if (gm_fabs(x) < 0.126)
            *sp = gm_taylor_sin(x, 0.0);
        else
            *sp = gm_copysign(gm_do_sin(gm_fabs(x), x > 0.0 ? 0.0 : -0.0), x);
        *cp = gm_do_cos(gm_fabs(x), x >= 0.0 ? 0.0 : -0.0);
    } else if (k < 0x400368fdu) {
        const double t = GM_SUB(GM_HP0, gm_fabs(x));
        *sp = gm_copysign(gm_do_cos(gm_fabs(t), t >= 0.0 ? GM_HP1 : -GM_HP1), x);
        const double a = GM_ADD(t, GM_HP1);
        const double da = GM_ADD(GM_SUB(t, a), GM_HP1);
        *cp = gm_fabs(a) < 0.126 ? gm_taylor_sin(a, da)
                                 : gm_copysign(gm_do_sin(gm_fabs(a), a <= 0.0 ? gm_neg(da) : da), a);
    } else if (k < 0x419921fbu) {
        double b, db;
        const int n = gm_reduce(x, b, db);
        *sp = gm_sincos_reduced(b, db, n);
        *cp = gm_sincos_reduced(b, db, n + 1);
    } else {
        *sp = gm_sin(x);
        *cp = gm_cos(x);
    }
}

// ---- the same sin/cos pair without divergence (the transport's form) -----
// Every branch of gm_sin / gm_cos ends in one of three evaluations -- do_sin
// (or its Taylor form below 0.126), do_cos -- of a prepared argument, then a
// sign fix.  Here each lane prepares both arguments with selects, and one
// select-driven evaluator serves both kinds: the operations each lane's
// value goes through are exactly those of gm_sin / gm_cos (bit-identical by
// construction and checked), but a warp no longer runs every branch its
// lanes' angles touch (the ranges split ~14/25/61% over (0, 2 pi]).
GM_HD double gm_eval_kind(double a, double da, bool is_cos) {
    const double xa = gm_fabs(a);
    const double dx = (is_cos ? a < 0.0 : a <= 0.0) ? gm_neg(da) : da;
    const double u = GM_ADD(xa, GM_BIG);
    const double x0 = GM_SUB(xa, GM_SUB(u, GM_BIG));
    const double x = is_cos ? GM_ADD(x0, dx) : x0;
    const int k4 = (int)((uint32_t)gm_bits(u) << 2);
    const double xx = GM_MUL(x, x);
    const double p = GM_FMA(xx, GM_SN5, GM_SN3);
    const double xxx = GM_MUL(x, xx);
    const double s = is_cos ? GM_FMA(xxx, p, x) : GM_ADD(x, GM_FMA(xxx, p, dx));
    const double pcx = GM_MUL(xx, GM_FMA(xx, GM_FMA(xx, GM_CS6, GM_CS4), 0.5));
    const double c = is_cos ? pcx : GM_FMA(x, dx, pcx);
    const double sn = GM_SC(k4, 0), ssn = GM_SC(k4, 1), cs = GM_SC(k4, 2), ccs = GM_SC(k4, 3);
    // do_sin: sn + (s cs + (-c sn + (s ccs + ssn)))
    // do_cos: cs + (-s sn + (-c cs + (-s ssn + ccs)))
    const double t1 = is_cos ? gm_neg(sn) : cs, t2 = is_cos ? cs : sn;
    const double t3 = is_cos ? gm_neg(ssn) : ccs, t4 = is_cos ? ccs : ssn;
    const double cor = GM_FMA(s, t1, GM_FMA(-c, t2, GM_FMA(s, t3, t4)));
    const double r = GM_ADD(t2, cor);
    if (is_cos) return r;
    // do_sin's Taylor form for |a| < 0.126 (a and da as given)
    return xa < 0.126 ? gm_taylor_sin(a, da) : gm_copysign(r, a);
}

GM_HD void gm_sincos_simt(double x, double* sp, double* cp) {
    const uint32_t k = (uint32_t)(gm_bits(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e500000u || k >= 0x419921fbu) {  // tiny or huge: the branchy form
        gm_sincos(x, sp, cp);
        return;
    }
    const double ax = gm_fabs(x);
    // range M (0.855469 <= |x| < 2.426265): t = hp0 - |x|
    const double t = GM_SUB(GM_HP0, ax);
    const double am = GM_ADD(t, GM_HP1);
    const double dam = GM_ADD(GM_SUB(t, am), GM_HP1);
    // range R: x = n pi/2 + b + db
    double b, db;
    const int n = gm_reduce(x, b, db);
    const bool rd = k < 0x3feb6000u, rm = !rd && k < 0x400368fdu;
    // sin: D do_sin(x, 0); M do_cos(t, hp1) with copysign(., x); R by n
    const bool s_cos = rm || (!rd && (n & 1));
    const double s_a = rd ? x : rm ? t : b;
    const double s_da = rd ? 0.0 : rm ? GM_HP1 : db;
    // cos: D do_cos(x, 0); M do_sin(am, dam); R by n + 1
    const bool c_cos = rd || (!rm && !(n & 1));
    const double c_a = rd ? x : rm ? am : b;
    const double c_da = rd ? 0.0 : rm ? dam : db;
    double sv = gm_eval_kind(s_a, s_da, s_cos);
    double cv = gm_eval_kind(c_a, c_da, c_cos);
    if (rm) sv = gm_copysign(sv, x);
    if (!rd && !rm) {
        if (n & 2) sv = gm_neg(sv);
        if ((n + 1) & 2) cv = gm_neg(cv);
    }
    *sp = sv;
    *cp = cv;
}

#endif  // BT_GLIBC_MATH
