// ORACLE — test infrastructure only. Never linked into the product; only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
//
// liboracle.so: the CPU restatement of the reference's OuroMamba-Quant
// inference path (oracle/oracle_ops.hpp) driven by the shared model driver
// (oracle/driver.hpp), behind the C API of oracle/capi_impl.hpp.
// Parity status: pinned bit-for-bit against the reference's own compiled code
// (oracle/_ref, tests/test_oracle_pin.py) and its committed golden vectors
// (tests/golden/, made by tests/golden/make_golden.py).
#include "oracle_ops.hpp"

namespace oro {

struct OracleOps {
    using State = OutlierState;
    struct Weight {
        const std::int8_t* codes = nullptr;
        const double* scales = nullptr;
        std::size_t rows = 0, cols = 0;
    };
    struct Prepared;

    static ModelW make_model(const Dims& d, const std::vector<int>& orders, std::uint64_t seed) {
        return make_toy_model(d, orders, seed);
    }
    static QRows quantize_rows(const std::vector<double>& w, std::size_t rows, unsigned bits) {
        return oro::quantize_rows(w, rows, bits);
    }
    static void mm_nt(const double* a, const double* b, double* c, std::size_t m, std::size_t k, std::size_t n) {
        oro::mm_nt(a, b, c, m, k, n);
    }
    static double softplus(double x) { return softplus_val(x); }
    static double silu(double x) { return silu_val(x); }
    static void refresh(State& st, std::size_t t, std::size_t n) { maybe_refresh(st, t, n); }
    static bool detect(State& st, const double* x, std::size_t e, std::size_t n, double th, double s, unsigned b) {
        return detect_outliers(st, x, e, n, th, s, b);
    }
    static void fake_quant(double* x, std::size_t e, std::size_t n, const State* st, double s, unsigned ab,
                           unsigned ob) {
        fake_quant_step(x, e, n, st, s, ab, ob);
    }
    static std::vector<std::size_t> list(const State& st, std::size_t) { return st.list(); }
    static SplitOperands split(const double* x, std::size_t k, std::size_t c, const std::vector<std::size_t>& o,
                               double s, unsigned ab, unsigned ob) {
        return split_quantize(x, k, c, o, s, ab, ob);
    }
    static GemmResult hybrid(const Weight& w, const SplitOperands& sp, double s) {
        return hybrid_gemm(w.codes, w.scales, w.rows, w.cols, sp.inlier_codes.data(), sp.outliers.cols ? sp.outliers.cols : 1,
                           s, sp.outliers);
    }
    static GemmResult hybrid_raw(const std::int8_t* w, const double* ws, std::size_t m, std::size_t k,
                                 const std::int8_t* x, std::size_t c, double s, const OutlierBuffer& ob) {
        return hybrid_gemm(w, ws, m, k, x, c, s, ob);
    }
    static std::vector<std::uint8_t> pack(const std::int8_t* codes, std::size_t r, std::size_t c) {
        return pack_int4(codes, r, c);
    }
    template <class Q>
    static Prepared prepare(const Q& q);
};

}  // namespace oro

#include "driver.hpp"

namespace oro {
struct OracleOps::Prepared {
    struct Blk {
        Weight in, out;
        std::vector<Weight> xp;
    };
    std::vector<Blk> blocks;
};
template <class Q>
OracleOps::Prepared OracleOps::prepare(const Q& q) {
    auto mk = [](const QRows& r) {
        Weight w;
        w.codes = r.codes.data();
        w.scales = r.scales.data();
        w.rows = r.scales.size();
        w.cols = r.codes.size() / w.rows;
        return w;
    };
    Prepared p;
    for (const auto& b : q.blocks) {
        Prepared::Blk pb;
        pb.in = mk(b.in);
        pb.out = mk(b.out);
        for (const auto& x : b.xp) pb.xp.push_back(mk(x));
        p.blocks.push_back(std::move(pb));
    }
    return p;
}
}  // namespace oro

using OPS = oro::OracleOps;
#include "capi_impl.hpp"
