// Self-test of csrc/glibc_math.cuh (host build) against the C library:
// gm_log / gm_sin / gm_cos must equal libm's log / sin / cos bit for bit on
// the transport's arguments (log on (0, 1], sin/cos on (0, 2 pi]) and around
// every branch threshold of the three algorithms.
//   glibc_math_selftest N SEED  ->  prints "checked <n> mismatches <m>" per function
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include "glibc_math.cuh"

#if !BT_GLIBC_MATH
int main() { std::printf("unavailable\n"); return 0; }
#else
static uint64_t st;
static uint64_t next() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
static double unit() { return ((double)(next() >> 11) + 1.0) * (1.0 / 9007199254740992.0); }
static bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
    st = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 88172645463325252ull;
    // the libm entry points themselves (no compiler builtins or constant folding)
    void* m = dlopen("libm.so.6", RTLD_NOW);
    if (!m) return 2;
    auto lg = reinterpret_cast<double (*)(double)>(dlsym(m, "log"));
    auto sn = reinterpret_cast<double (*)(double)>(dlsym(m, "sin"));
    auto cs = reinterpret_cast<double (*)(double)>(dlsym(m, "cos"));
    long bad[3] = {0, 0, 0}, cnt[3] = {0, 0, 0};
    auto check = [&](int f, double x) {
        double a = f == 0 ? gm_log(x) : f == 1 ? gm_sin(x) : gm_cos(x);
        const double b = f == 0 ? lg(x) : f == 1 ? sn(x) : cs(x);
        if (f > 0) {  // gm_sincos and gm_sincos_simt must give the same pair
            double s2, c2, s3, c3;
            gm_sincos(x, &s2, &c2);
            gm_sincos_simt(x, &s3, &c3);
            if (!same(f == 1 ? s2 : c2, a)) a = f == 1 ? s2 : c2;
            if (!same(f == 1 ? s3 : c3, a)) a = f == 1 ? s3 : c3;
        }
        ++cnt[f];
        if (!same(a, b)) {
            if (bad[f] < 5) std::printf("mismatch f=%d x=%a got %a want %a\n", f, x, a, b);
            ++bad[f];
        }
    };
    const double two_pi = 2.0 * 3.141592653589793;
    for (long i = 0; i < n; ++i) {
        const double u = unit();
        check(0, u);                                  // the flight's log(u), u in (0, 1]
        check(0, 0.9375 + 0.125 * unit());            // log's near-1 branch
        check(1, two_pi * u);                         // the scatter angle
        check(2, two_pi * u);
    }
    // branch thresholds and their neighbourhoods (both functions)
    const double edges[] = {0.126, 0.855469, 2.426265, 3.141592653589793 / 2, 3.141592653589793,
                            3 * 3.141592653589793 / 2, two_pi, 0x1p-26, 0x1p-27, 1e-3};
    for (double e : edges)
        for (int k = -2000; k <= 2000; ++k) {
            const double x = e * (1.0 + k * 1e-13);
            check(1, x);
            check(2, x);
            double y = e;
            for (int j = 0; j < (k < 0 ? -k : k) % 64; ++j) y = std::nextafter(y, k < 0 ? 0.0 : 10.0);
            check(1, y);
            check(2, y);
        }
    for (double x = 0x1p-53; x <= 1.0; x *= 1.0009765625) check(0, x);
    check(0, 1.0);
    const char* name[3] = {"log", "sin", "cos"};
    for (int f = 0; f < 3; ++f) std::printf("%s checked %ld mismatches %ld\n", name[f], cnt[f], bad[f]);
    return (bad[0] || bad[1] || bad[2]) ? 1 : 0;
}
#endif
