// Checks the device exp/log1p restatement (paper_2503_10959_b200/csrc/glibc_math.cuh,
// compiled here for the host without contraction) against the live libm, which is
// what the reference's std::exp/std::log1p call. Prints one line per range:
// "<name> <mismatches> <samples>". Built and run by tests/test_glibc_math.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "glibc_math.cuh"

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
    std::mt19937_64 g(20250318);
    struct Range {
        const char* name;
        double lo, hi;
        int fn;
    } ranges[] = {
        {"exp_scan[-60,0]", -60, 0, 0},      {"exp[-1,1]", -1, 1, 0},          {"exp[-745,710]", -745, 710, 0},
        {"exp_tiny", -1e-10, 1e-10, 0},      {"exp_subnormal", -760, -700, 0}, {"exp_overflow", 500, 710, 0},
        {"log1p_softplus(0,1]", 0, 1, 1},    {"log1p[-1,10]", -1, 10, 1},      {"log1p_small", 0, 1e-6, 1},
        {"log1p_edge", 0.40, 0.43, 1},       {"log1p_neg", -0.3, -0.28, 1},    {"log1p_huge", 1e15, 1e17, 1},
        {"log1p_tiny", 1e-9, 1e-8, 1},
    };
    for (const Range& r : ranges) {
        std::uniform_real_distribution<double> d(r.lo, r.hi);
        long bad = 0;
        for (long i = 0; i < n; ++i) {
            const double x = d(g);
            const double a = r.fn ? ob::gl::log1p(x) : ob::gl::exp(x);
            const double b = r.fn ? std::log1p(x) : std::exp(x);
            bad += std::memcmp(&a, &b, sizeof a) != 0;
        }
        std::printf("%s %ld %ld\n", r.name, bad, n);
    }
    // log1p where 1 + x sits near a power of two (the |f| < 2^-20 branches)
    long bad = 0, cnt = 0;
    for (int e = -60; e < 60; ++e)
        for (int j = -2000; j < 2000; ++j, ++cnt) {
            const double x = std::ldexp(1.0, e) - 1.0 + j * std::ldexp(1.0, e - 52);
            const double a = ob::gl::log1p(x), b = std::log1p(x);
            bad += std::memcmp(&a, &b, sizeof a) != 0;
        }
    std::printf("log1p_pow2 %ld %ld\n", bad, cnt);
    // special values
    const double sp[] = {0.0, -0.0, INFINITY, -INFINITY, NAN, 709.782712893384, 709.7827128933841, -745.1332191019411,
                         -745.1332191019412, -708.3964185322641, 1e-300, -1.0, -1.0 + 1e-16, 2e-54, 5e-324};
    bad = 0;
    for (double x : sp) {
        const double a = ob::gl::exp(x), b = std::exp(x), c = ob::gl::log1p(x), e = std::log1p(x);
        bad += (std::memcmp(&a, &b, sizeof a) != 0 && !(std::isnan(a) && std::isnan(b))) +
               (std::memcmp(&c, &e, sizeof c) != 0 && !(std::isnan(c) && std::isnan(e)));
    }
    std::printf("special %ld %zu\n", bad, sizeof sp / sizeof sp[0]);
    return 0;
}
