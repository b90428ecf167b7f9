// Host check of paper_1904_00429_b200/csrc/mlsk_libm.cuh against the system
// libm (glibc, whose ifunc picks the FMA variants on FMA/AVX2 CPUs): bit-exact
// comparison over random arguments in every branch of log / sin / cos.
//   libm_check <n per range> <seed>  -> one line per range: name n mismatches max_ulp
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "../../paper_1904_00429_b200/csrc/mlsk_libm.cuh"

static uint64_t bits(double x) { uint64_t b; std::memcpy(&b, &x, 8); return b; }
static double from(uint64_t b) { double d; std::memcpy(&d, &b, 8); return d; }

template <class F, class G>
static int run(const char* name, long n, std::mt19937_64& rng, G gen, F mine, double (*ref)(double)) {
    long bad = 0;
    long long worst = 0;
    double where = 0;
    for (long i = 0; i < n; ++i) {
        const double x = gen(rng);
        const double a = mine(x), b = ref(x);
        if (bits(a) != bits(b) && !(std::isnan(a) && std::isnan(b))) {
            ++bad;
            long long d = (long long)bits(a) - (long long)bits(b);
            if (d < 0) d = -d;
            if (d > worst) { worst = d; where = x; }
        }
    }
    std::printf("%s %ld %ld %lld %.17g\n", name, n, bad, worst, where);
    return bad != 0;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
    std::mt19937_64 rng(argc > 2 ? std::strtoull(argv[2], 0, 10) : 1);
    auto u01 = [](std::mt19937_64& r) { return (double)(r() >> 11) * 0x1.0p-53; };  // rng.hpp uniform01
    auto upos = [&](std::mt19937_64& r) { return 1.0 - u01(r); };                   // rng.hpp uniform_pos
    auto anybits = [](std::mt19937_64& r) {  // any positive finite double
        for (;;) { double x = from(r() & 0x7fffffffffffffffull); if (std::isfinite(x)) return x; } };
    auto range = [&](double lo, double hi) {
        return [=](std::mt19937_64& r) { double u = (double)(r() >> 11) * 0x1.0p-53; double x = lo + (hi - lo) * u;
                                          return (r() & 1) ? -x : x; }; };
    auto logrange = [&](double lo, double hi) {  // log-uniform magnitude, random sign
        return [=](std::mt19937_64& r) { double u = (double)(r() >> 11) * 0x1.0p-53;
                                          double x = std::exp(std::log(lo) + (std::log(hi) - std::log(lo)) * u);
                                          return (r() & 1) ? -x : x; }; };
    auto L = [](double x) { return mlsk_libm::log(x); };
    auto S = [](double x) { return mlsk_libm::sin(x); };
    auto C = [](double x) { return mlsk_libm::cos(x); };
    auto theta = [&](std::mt19937_64& r) { return 6.283185307179586 * u01(r); };   // Box-Muller angle
    int fails = 0;
    fails += run("log_upos", n, rng, upos, L, ::log);
    fails += run("log_near1", n, rng, [](std::mt19937_64& r) { return 0.9375 + 0.13 * (double)(r() >> 11) * 0x1.0p-53; }, L, ::log);
    fails += run("log_anybits", n, rng, anybits, L, ::log);
    fails += run("log_subnormal", n / 10, rng, [](std::mt19937_64& r) { return from(r() & 0x000fffffffffffffull); }, L, ::log);
    fails += run("sin_theta", n, rng, theta, S, ::sin);
    fails += run("cos_theta", n, rng, theta, C, ::cos);
    fails += run("sin_tiny", n / 10, rng, logrange(1e-12, 0.126), S, ::sin);
    fails += run("cos_tiny", n / 10, rng, logrange(1e-12, 0.126), C, ::cos);
    fails += run("sin_0_0.86", n, rng, range(0.0, 0.86), S, ::sin);
    fails += run("cos_0_0.86", n, rng, range(0.0, 0.86), C, ::cos);
    fails += run("sin_0.85_2.43", n, rng, range(0.85, 2.43), S, ::sin);
    fails += run("cos_0.85_2.43", n, rng, range(0.85, 2.43), C, ::cos);
    fails += run("sin_2.4_1e3", n, rng, logrange(2.4, 1e3), S, ::sin);
    fails += run("cos_2.4_1e3", n, rng, logrange(2.4, 1e3), C, ::cos);
    fails += run("sin_1e3_1e8", n, rng, logrange(1e3, 1.05e8), S, ::sin);
    fails += run("cos_1e3_1e8", n, rng, logrange(1e3, 1.05e8), C, ::cos);
    return fails ? 1 : 0;
}
