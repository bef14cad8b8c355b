// ORACLE — test infrastructure only. Never linked into the product.
//
// CPU restatement of the reference's hot-path primitives (OuroMamba-Quant,
// /root/reference/proj/src/ouro/*). Every function cites the reference
// file:line it restates. Arithmetic is IEEE f64 in the reference's operation
// order; the build uses -ffp-contract=off as the reference does
// (CMakeLists.txt:19-21), so results are bit-identical to the reference's own
// code compiled here (pinned by tests/test_oracle_pin.py against oracle/_ref).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace oro {

struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
inline void require(bool c, const char* m) {
    if (!c) throw ValidationError(m);
}

// ---- RNG: SeededRng, rng.hpp:13-40 / rng.cpp:7-50 ---------------------------
class Rng {
  public:
    explicit Rng(std::uint64_t seed) : gen_(seed), seed_(seed) {}
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }  // rng.cpp:7-9
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }  // rng.cpp:11-13
    double normal() {  // Box-Muller with cached spare, rng.cpp:15-27
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = 1.0 - uniform();
        double u2 = uniform();
        double r = std::sqrt(-2.0 * std::log(u1));
        double a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }
    double normal(double mean, double sd) { return mean + sd * normal(); }  // rng.hpp:25
    std::uint64_t below(std::uint64_t n) {  // rejection sampling, rng.cpp:29-37
        std::uint64_t limit = UINT64_MAX - UINT64_MAX % n, v;
        do v = gen_(); while (v >= limit);
        return v % n;
    }
    Rng fork(std::uint64_t salt) const {  // SplitMix64 finalizer, rng.cpp:43-49
        std::uint64_t z = seed_ + 0x9e3779b97f4a7c15ull * (salt + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return Rng(z ^ (z >> 31));
    }

  private:
    std::mt19937_64 gen_;
    std::uint64_t seed_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

// ---- scalar kernels: tensor.hpp:146-154 ------------------------------------
inline double sigmoid_val(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
    double e = std::exp(x);
    return e / (1.0 + e);
}
inline double softplus_val(double x) { return std::max(x, 0.0) + std::log1p(std::exp(-std::fabs(x))); }
inline double silu_val(double x) { return x * sigmoid_val(x); }

// c (m x n) = a (m x k) . b^T with b stored n x k; the (!ta, tb) branch of
// detail::mm, tensor.cpp:373-382: per output a k-ascending sum from 0.0,
// then added into the zero-filled output.
inline void mm_nt(const double* a, const double* b, double* c, std::size_t m, std::size_t k,
                  std::size_t n) {
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j) {
            double s = 0.0;
            const double* ar = a + i * k;
            const double* br = b + j * k;
            for (std::size_t p = 0; p < k; ++p) s += ar[p] * br[p];
            c[i * n + j] = 0.0 + s;
        }
}

// ---- quantization primitives: quant.cpp:15-42 ------------------------------
inline double qmax_for(unsigned bits) {
    require(bits >= 2 && bits <= 62, "bit width must be in [2, 62]");
    return static_cast<double>((std::int64_t{1} << (bits - 1)) - 1);
}
inline std::int64_t quantize_code(double x, double s, unsigned bits) {  // quant.cpp:29-35
    double q = qmax_for(bits);
    double r = std::round(x / s);  // half away from zero
    if (r > q) r = q;
    if (r < -q) r = -q;
    return static_cast<std::int64_t>(r);
}
inline double scale_for(const double* x, std::size_t n, unsigned bits) {  // quant.cpp:37-42
    double mx = 0.0;
    for (std::size_t i = 0; i < n; ++i) mx = std::max(mx, std::fabs(x[i]));
    if (mx == 0.0) return 1.0;
    return mx / qmax_for(bits);
}

// Outlier bookkeeping, quant.hpp:60-65. A per-channel flag vector is the same
// set as the reference's sorted o_list; iteration in ascending channel order
// reproduces its order.
struct OutlierState {
    std::vector<char> in;
    std::size_t steps_since_refresh = 0;
    void ensure(std::size_t e) {
        if (in.size() != e) in.assign(e, 0);
    }
    std::vector<std::size_t> list() const {
        std::vector<std::size_t> v;
        for (std::size_t i = 0; i < in.size(); ++i)
            if (in[i]) v.push_back(i);
        return v;
    }
};

inline bool maybe_refresh(OutlierState& st, std::size_t t, std::size_t n_refresh) {  // quant.cpp:303-311
    if (n_refresh == 0 || t == 0 || t % n_refresh != 0) {
        if (t > 0) ++st.steps_since_refresh;
        return false;
    }
    std::fill(st.in.begin(), st.in.end(), 0);
    st.steps_since_refresh = 0;
    return true;
}

// detect_outliers, quant.cpp:313-335 (channel = row of n values). Returns
// DetectResult::scanned.
inline bool detect_outliers(OutlierState& st, const double* x, std::size_t e, std::size_t n,
                            double theta, double scale_inlier, unsigned act_bits) {
    st.ensure(e);
    double mx = 0.0;
    for (std::size_t ch = 0; ch < e; ++ch) {
        if (st.in[ch]) continue;
        for (std::size_t s = 0; s < n; ++s) mx = std::max(mx, std::fabs(x[ch * n + s]));
    }
    double s_dyn = mx / qmax_for(act_bits);
    if (s_dyn <= scale_inlier) return false;
    for (std::size_t ch = 0; ch < e; ++ch) {
        double peak = 0.0;
        for (std::size_t s = 0; s < n; ++s) peak = std::max(peak, std::fabs(x[ch * n + s]));
        if (peak > theta && !st.in[ch]) st.in[ch] = 1;
    }
    return true;
}

// fake_quant_step, quant.cpp:337-351 (in place).
inline void fake_quant_step(double* x, std::size_t e, std::size_t n, const OutlierState* st,
                            double scale_inlier, unsigned act_bits, unsigned outlier_bits) {
    for (std::size_t ch = 0; ch < e; ++ch) {
        double* row = x + ch * n;
        if (st && ch < st->in.size() && st->in[ch]) {
            double s = scale_for(row, n, outlier_bits);
            for (std::size_t i = 0; i < n; ++i)
                row[i] = static_cast<double>(quantize_code(row[i], s, outlier_bits)) * s;
        } else {
            for (std::size_t i = 0; i < n; ++i)
                row[i] = static_cast<double>(quantize_code(row[i], scale_inlier, act_bits)) * scale_inlier;
        }
    }
}

// ---- hybrid GEMM operands: gemm.hpp:20-57 / gemm.cpp:54-135 ----------------
struct OutlierBuffer {
    std::vector<std::size_t> channels;
    std::vector<std::int8_t> codes;  // channels.size() x cols
    std::vector<double> scales;
    std::size_t cols = 0;
};
struct SplitOperands {
    std::vector<std::int8_t> inlier_codes;  // k x c
    OutlierBuffer outliers;
};

inline SplitOperands split_quantize(const double* x, std::size_t k, std::size_t c,
                                    const std::vector<std::size_t>& o_list, double inlier_scale,
                                    unsigned act_bits, unsigned outlier_bits) {  // gemm.cpp:106-135
    require(inlier_scale > 0.0, "split_quantize: inlier scale must be positive");
    SplitOperands out;
    out.inlier_codes.assign(k * c, 0);
    out.outliers.cols = c;
    out.outliers.channels = o_list;
    out.outliers.scales.resize(o_list.size());
    out.outliers.codes.resize(o_list.size() * c);
    std::size_t j = 0;
    for (std::size_t ch = 0; ch < k; ++ch) {
        const double* row = x + ch * c;
        if (j < o_list.size() && o_list[j] == ch) {
            require(j == 0 || o_list[j - 1] < ch, "split_quantize: channels must strictly increase");
            double s = scale_for(row, c, outlier_bits);
            out.outliers.scales[j] = s;
            for (std::size_t i = 0; i < c; ++i)
                out.outliers.codes[j * c + i] = static_cast<std::int8_t>(quantize_code(row[i], s, outlier_bits));
            ++j;
        } else {
            for (std::size_t i = 0; i < c; ++i)
                out.inlier_codes[ch * c + i] = static_cast<std::int8_t>(quantize_code(row[i], inlier_scale, act_bits));
        }
    }
    require(j == o_list.size(), "split_quantize: channel index out of range");
    return out;
}

// pack_int4, gemm.cpp:60-76: two codes per byte, low nibble = even column.
inline std::vector<std::uint8_t> pack_int4(const std::int8_t* codes, std::size_t rows, std::size_t cols) {
    std::size_t stride = (cols + 1) / 2;
    std::vector<std::uint8_t> bytes(rows * stride, 0);
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t c = 0; c < cols; ++c) {
            std::int8_t v = codes[r * cols + c];
            require(v >= -7 && v <= 7, "pack_int4: code outside [-7, 7]");
            std::uint8_t nib = static_cast<std::uint8_t>(v) & 0x0F;
            std::uint8_t& b = bytes[r * stride + c / 2];
            b = (c & 1) ? static_cast<std::uint8_t>(b | (nib << 4)) : static_cast<std::uint8_t>(b | nib);
        }
    return bytes;
}

struct GemmResult {
    std::vector<std::int32_t> acc_inlier, acc_outlier;
    std::vector<double> output;
};

// hybrid_gemm, gemm.cpp:181-225, generalised to int8 inlier codes (the
// reference packs A4 inliers; its A8 inlier oracle is the triple loop of
// tests/test_gemm.cpp:25-35). w: m x k codes (row = output), x: k x c codes.
inline GemmResult hybrid_gemm(const std::int8_t* w, const double* w_scales, std::size_t m,
                              std::size_t k, const std::int8_t* x_inlier, std::size_t c,
                              double inlier_scale, const OutlierBuffer& outliers) {
    require(inlier_scale > 0.0, "hybrid_gemm: inlier scale must be positive");
    require(outliers.scales.size() == outliers.channels.size(), "hybrid_gemm: one scale per outlier channel");
    GemmResult r;
    r.acc_inlier.assign(m * c, 0);
    r.acc_outlier.assign(m * c, 0);
    r.output.assign(m * c, 0.0);
    for (std::size_t row = 0; row < m; ++row)  // gemm_i4, gemm.cpp:137-158 (exact int32)
        for (std::size_t kk = 0; kk < k; ++kk) {
            std::int32_t wv = w[row * k + kk];
            for (std::size_t col = 0; col < c; ++col)
                r.acc_inlier[row * c + col] += wv * x_inlier[kk * c + col];
        }
    std::size_t n_o = outliers.channels.size();
    for (std::size_t row = 0; row < m; ++row) {  // fused epilogue, gemm.cpp:201-222
        const std::int32_t* ain = r.acc_inlier.data() + row * c;
        std::int32_t* aout = r.acc_outlier.data() + row * c;
        double* orow = r.output.data() + row * c;
        for (std::size_t col = 0; col < c; ++col) orow[col] = inlier_scale * static_cast<double>(ain[col]);
        for (std::size_t j = 0; j < n_o; ++j) {
            std::int32_t wv = w[row * k + outliers.channels[j]];
            double coeff = outliers.scales[j] * static_cast<double>(wv);
            const std::int8_t* xrow = outliers.codes.data() + j * c;
            for (std::size_t col = 0; col < c; ++col) {
                aout[col] += wv * xrow[col];
                orow[col] += coeff * static_cast<double>(xrow[col]);
            }
        }
        double ws = w_scales[row];
        for (std::size_t col = 0; col < c; ++col) orow[col] = ws * orow[col];
    }
    return r;
}

// ---- model structure ---------------------------------------------------------
struct Dims {  // ModelDims, ssm.hpp:42-56
    std::size_t image = 32, channels = 3, patch = 4, embed = 16, state = 4, blocks = 2, classes = 10,
                conv_width = 3;
    std::size_t grid() const { return image / patch; }
    std::size_t tokens() const { return grid() * grid(); }
    std::size_t patch_vals() const { return patch * patch * channels; }
};
struct DirW {
    std::vector<double> a, w_b, w_c, w_delta, b_delta;  // E x N, N x E, N x E, E x E, E
};
struct BlockW {
    std::vector<double> w_in, w_gate, conv, out_proj;  // E x E, E x E, E x W, E x E
    std::vector<DirW> dirs;
};
struct ModelW {
    Dims d;
    std::vector<int> orders;  // ScanOrder values: 0 row-fwd, 1 row-bwd, 2 col-fwd, 3 col-bwd
    std::vector<double> patch_w, patch_b, head_w, head_b;
    std::vector<BlockW> blocks;
};

// scan_permutation, ssm.cpp:30-46: perm[t] = canonical token at scan step t.
inline std::vector<std::size_t> scan_permutation(int order, std::size_t grid) {
    std::size_t m = grid * grid;
    std::vector<std::size_t> perm(m);
    for (std::size_t t = 0; t < m; ++t) {
        std::size_t fast = t % grid, slow = t / grid, canon = 0;
        switch (order) {
            case 0: canon = slow * grid + fast; break;
            case 1: canon = m - 1 - (slow * grid + fast); break;
            case 2: canon = fast * grid + slow; break;
            case 3: canon = m - 1 - (fast * grid + slow); break;
            default: throw ValidationError("unknown scan order value");
        }
        perm[t] = canon;
    }
    return perm;
}

// patch_gather_indices, ssm.cpp:72-84.
inline std::vector<std::size_t> patch_gather_indices(const Dims& d) {
    std::vector<std::size_t> idx;
    idx.reserve(d.tokens() * d.patch_vals());
    std::size_t g = d.grid();
    for (std::size_t gr = 0; gr < g; ++gr)
        for (std::size_t gc = 0; gc < g; ++gc)
            for (std::size_t pr = 0; pr < d.patch; ++pr)
                for (std::size_t pc = 0; pc < d.patch; ++pc)
                    for (std::size_t ch = 0; ch < d.channels; ++ch)
                        idx.push_back(((gr * d.patch + pr) * d.image + gc * d.patch + pc) * d.channels + ch);
    return idx;
}

// make_toy_model, ssm.cpp:88-120 (draw order: patch_embed, head, then per
// block w_in, w_gate, conv, out_proj, then per dir a, w_b, w_c, w_delta).
inline std::vector<double> gaussian(Rng& rng, std::size_t n, std::size_t fan_in) {  // ssm.cpp:64-69
    std::vector<double> t(n);
    double s = 1.0 / std::sqrt(static_cast<double>(fan_in));
    for (double& v : t) v = rng.normal(0.0, s);
    return t;
}
inline ModelW make_toy_model(const Dims& d, const std::vector<int>& orders, std::uint64_t seed) {
    require(d.patch >= 1 && d.image >= d.patch && d.image % d.patch == 0,
            "image side must be a positive multiple of the patch side");  // ssm.cpp:54-60
    require(!orders.empty(), "model needs at least one scan order");
    ModelW m;
    m.d = d;
    m.orders = orders;
    Rng rng(seed);
    std::size_t e = d.embed, n = d.state;
    m.patch_w = gaussian(rng, e * d.patch_vals(), d.patch_vals());
    m.patch_b.assign(e, 0.0);
    m.head_w = gaussian(rng, d.classes * e, e);
    m.head_b.assign(d.classes, 0.0);
    for (std::size_t b = 0; b < d.blocks; ++b) {
        BlockW blk;
        blk.w_in = gaussian(rng, e * e, e);
        blk.w_gate = gaussian(rng, e * e, e);
        blk.conv = gaussian(rng, e * d.conv_width, d.conv_width);
        blk.out_proj = gaussian(rng, e * e, e);
        for (std::size_t k = 0; k < orders.size(); ++k) {
            DirW p;
            p.a.resize(e * n);
            for (double& v : p.a) v = -std::exp(rng.uniform(0.0, 1.0));
            p.w_b = gaussian(rng, n * e, e);
            p.w_c = gaussian(rng, n * e, e);
            p.w_delta = gaussian(rng, e * e, e);
            p.b_delta.assign(e, 0.0);
            blk.dirs.push_back(std::move(p));
        }
        m.blocks.push_back(std::move(blk));
    }
    return m;
}

// quantize_weights + dequantize_rows, quant.cpp:355-382.
struct QRows {
    std::vector<std::int8_t> codes;
    std::vector<double> scales;
    std::vector<double> deq;
};
inline QRows quantize_rows(const std::vector<double>& w, std::size_t rows, unsigned bits) {
    QRows q;
    std::size_t cols = w.size() / rows;
    q.codes.resize(w.size());
    q.scales.resize(rows);
    q.deq.resize(w.size());
    for (std::size_t r = 0; r < rows; ++r) {
        const double* row = w.data() + r * cols;
        double s = scale_for(row, cols, bits);
        q.scales[r] = s;
        for (std::size_t c = 0; c < cols; ++c)
            q.codes[r * cols + c] = static_cast<std::int8_t>(quantize_code(row[c], s, bits));
    }
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t c = 0; c < cols; ++c)
            q.deq[r * cols + c] = static_cast<double>(q.codes[r * cols + c]) * q.scales[r];
    return q;
}

// Linearly interpolated quantile, quant.cpp:117-125 (internal there).
inline double quantile(std::vector<double> v, double q) {
    require(!v.empty(), "quantile of empty set");
    std::sort(v.begin(), v.end());
    double pos = q * static_cast<double>(v.size() - 1);
    std::size_t lo = static_cast<std::size_t>(pos);
    if (lo + 1 >= v.size()) return v.back();
    double frac = pos - static_cast<double>(lo);
    return v[lo] + frac * (v[lo + 1] - v[lo]);
}

}  // namespace oro
