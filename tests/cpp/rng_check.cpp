// The library's SeededRng (paper_2503_10959_b200/csrc/seeded_rng.h) against the
// reference's own (rng.cpp, compiled in oracle/_ref): uniform, uniform(lo, hi),
// normal (with the cached spare), below, fill_normal and fork produce the same
// values bit for bit. Prints "ok" or the first difference. Built by
// tests/test_seeded_rng.py (CPU).
#include <cstdio>
#include <cstring>
#include <vector>

#include "ouro/rng.hpp"
#include "seeded_rng.h"

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

int main() {
    for (unsigned long long seed : {0ull, 1ull, 1234ull, 0xdeadbeefcafef00dull}) {
        ouro::SeededRng r(seed);
        ob::SeededRng g(seed);
        for (int i = 0; i < 20000; ++i) {
            const int op = i % 5;
            if (op == 0 && !same(r.uniform(), g.uniform())) return std::printf("uniform differs at %d\n", i), 1;
            if (op == 1 && !same(r.uniform(-3.0, 0.5), g.uniform(-3.0, 0.5)))
                return std::printf("uniform(lo,hi) differs at %d\n", i), 1;
            if (op == 2 && !same(r.normal(), g.normal())) return std::printf("normal differs at %d\n", i), 1;
            if (op == 3) {
                const unsigned long long n = 1 + (i * 7919ull) % 1000003ull;
                if (r.below(n) != g.below(n)) return std::printf("below differs at %d\n", i), 1;
            }
            if (op == 4 && !same(r.normal(0.5, 2.0), g.normal(0.5, 2.0)))
                return std::printf("normal(mean,sd) differs at %d\n", i), 1;
        }
        std::vector<double> a(777), b(777);
        r.fill_normal(a, 0.0, 1.0);
        g.fill_normal(b, 0.0, 1.0);
        if (std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) != 0) return std::printf("fill_normal\n"), 1;
        for (unsigned long long salt : {0ull, 7ull, 99ull}) {
            ouro::SeededRng rf = r.fork(salt);
            ob::SeededRng gf = ob::SeededRng(seed).fork(salt);
            for (int i = 0; i < 100; ++i)
                if (!same(rf.uniform(), gf.uniform())) return std::printf("fork(%llu) differs\n", salt), 1;
        }
    }
    std::printf("ok\n");
    return 0;
}
