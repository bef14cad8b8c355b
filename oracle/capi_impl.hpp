// ORACLE — test infrastructure only. Never linked into the product.
//
// The C API both CPU checkers export (liboracle.so over OracleOps, the
// reference build _ref/libouro_ref.so over RefOps), so the Python checker
// (oracle/oracle.py) drives either through identical calls. Include after
// defining `using OPS = ...;`. Errors follow the reference C ABI: status 2 for
// validation failures (capi.cpp:18-37), message in oro_last_error().
#pragma once
#include <cstdio>
#include <map>
#include <memory>

#include "driver.hpp"

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

struct ModelH {
    oro::ModelW w;
};
struct CalibH {
    oro::Calib c;
};
struct TraceH {
    std::map<std::string, std::vector<char>> blobs;
};

template <class T>
void put(TraceH& th, const std::string& k, const std::vector<T>& v) {
    std::vector<char> b(v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
    th.blobs[k] = std::move(b);
}

std::vector<double>* model_tensor(oro::ModelW& m, const std::string& name) {
    if (name == "patch_w") return &m.patch_w;
    if (name == "patch_b") return &m.patch_b;
    if (name == "head_w") return &m.head_w;
    if (name == "head_b") return &m.head_b;
    unsigned b = 0, d = 0;
    char field[32];
    if (std::sscanf(name.c_str(), "block%u.dir%u.%31s", &b, &d, field) == 3) {
        if (b >= m.blocks.size() || d >= m.blocks[b].dirs.size()) return nullptr;
        oro::DirW& p = m.blocks[b].dirs[d];
        std::string f(field);
        if (f == "a") return &p.a;
        if (f == "w_b") return &p.w_b;
        if (f == "w_c") return &p.w_c;
        if (f == "w_delta") return &p.w_delta;
        if (f == "b_delta") return &p.b_delta;
        return nullptr;
    }
    if (std::sscanf(name.c_str(), "block%u.%31s", &b, field) == 2) {
        if (b >= m.blocks.size()) return nullptr;
        std::string f(field);
        if (f == "w_in") return &m.blocks[b].w_in;
        if (f == "w_gate") return &m.blocks[b].w_gate;
        if (f == "conv") return &m.blocks[b].conv;
        if (f == "out_proj") return &m.blocks[b].out_proj;
    }
    return nullptr;
}

oro::Spec make_spec(const unsigned* bits, std::size_t n_refresh, double rho) {
    oro::Spec s;
    s.wbits = bits[0];
    s.abits = bits[1];
    s.obits = bits[2];
    s.n_refresh = n_refresh;
    s.rho = rho;
    return s;
}

}  // namespace

extern "C" {

const char* oro_last_error(void) { return g_err.c_str(); }

// dims: image, channels, patch, embed, state, blocks, classes, conv_width
int oro_model_create(const std::size_t* dims, const int* orders, std::size_t ndirs, std::uint64_t seed,
                     void** out) {
    return guarded([&] {
        oro::Dims d;
        d.image = dims[0];
        d.channels = dims[1];
        d.patch = dims[2];
        d.embed = dims[3];
        d.state = dims[4];
        d.blocks = dims[5];
        d.classes = dims[6];
        d.conv_width = dims[7];
        auto h = std::make_unique<ModelH>();
        h->w = OPS::make_model(d, std::vector<int>(orders, orders + ndirs), seed);
        *out = h.release();
    });
}
void oro_model_free(void* m) { delete static_cast<ModelH*>(m); }

long oro_model_get(void* m, const char* name, double* out, std::size_t cap) {
    auto* v = model_tensor(static_cast<ModelH*>(m)->w, name);
    if (!v) return -1;
    if (out) std::memcpy(out, v->data(), std::min(cap, v->size()) * sizeof(double));
    return static_cast<long>(v->size());
}
int oro_model_set(void* m, const char* name, const double* in, std::size_t n) {
    return guarded([&] {
        auto* v = model_tensor(static_cast<ModelH*>(m)->w, name);
        oro::require(v && v->size() == n, "model_set: unknown tensor or size mismatch");
        std::memcpy(v->data(), in, n * sizeof(double));
    });
}

// W4 codes/scales of one fake-quantized weight matrix (quant.cpp:355-372):
// which = "patch", "head", "block<b>.in" (w_in rows then w_gate rows),
// "block<b>.conv", "block<b>.out", "block<b>.xp<d>" (w_delta, w_b, w_c rows).
long oro_model_qweight(void* m, unsigned bits, const char* which, std::int8_t* codes, double* scales,
                       std::size_t cap_codes, std::size_t cap_scales) {
    long n = -1;
    guarded([&] {
        oro::QModel q = oro::quantize_model<OPS>(static_cast<ModelH*>(m)->w, bits);
        std::string s(which);
        const oro::QRows* r = nullptr;
        unsigned b = 0, d = 0;
        if (s == "patch") r = &q.patch;
        else if (s == "head") r = &q.head;
        else if (std::sscanf(s.c_str(), "block%u.xp%u", &b, &d) == 2 && b < q.blocks.size() && d < q.blocks[b].xp.size()) r = &q.blocks[b].xp[d];
        else if (std::sscanf(s.c_str(), "block%u.", &b) == 1 && b < q.blocks.size()) {
            std::string f = s.substr(s.find('.') + 1);
            if (f == "in") r = &q.blocks[b].in;
            else if (f == "conv") r = &q.blocks[b].conv;
            else if (f == "out") r = &q.blocks[b].out;
        }
        oro::require(r != nullptr, "qweight: unknown weight");
        if (codes) std::memcpy(codes, r->codes.data(), std::min(cap_codes, r->codes.size()));
        if (scales) std::memcpy(scales, r->scales.data(), std::min(cap_scales, r->scales.size()) * sizeof(double));
        n = static_cast<long>(r->codes.size());
    });
    return n;
}

// SeededRng(seed).normal() x n — the image generator of init_noise_batch
// (datagen.cpp:124-128) and test_ssm.cpp:150-152.
void oro_normal_fill(std::uint64_t seed, double* out, std::size_t n) {
    oro::Rng r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.normal();
}

int oro_calibrate(void* m, const double* images, std::size_t B, const unsigned* bits, std::size_t n_refresh,
                  double rho, int d1, int d2, int threads, void** out) {
    return guarded([&] {
        auto h = std::make_unique<CalibH>();
        h->c = oro::calibrate<OPS>(static_cast<ModelH*>(m)->w, images, B, make_spec(bits, n_refresh, rho), d1 != 0,
                                   d2 != 0, threads);
        *out = h.release();
    });
}

// Empty calibration with the model's geometry, to be filled with oro_calib_set.
int oro_calib_new(void* m, const unsigned* bits, std::size_t n_refresh, double rho, int d1, int d2, void** out) {
    return guarded([&] {
        const oro::ModelW& w = static_cast<ModelH*>(m)->w;
        auto h = std::make_unique<CalibH>();
        oro::Calib& c = h->c;
        c.spec = make_spec(bits, n_refresh, rho);
        c.spec.validate();
        c.tokens = w.d.tokens();
        c.embed = w.d.embed;
        c.state = w.d.state;
        c.blocks = w.blocks.size();
        c.ndirs = w.orders.size();
        c.d1 = d1 != 0;
        c.d2 = d2 != 0;
        oro::TCal z;
        z.s_in.assign(c.tokens, 1.0);
        z.s_full.assign(c.tokens, 1.0);
        z.excluded.assign(c.embed, 0);
        c.scan.assign(c.blocks * c.ndirs * 3, z);
        if (c.d2) c.lin.assign(c.blocks * c.nsites(), z);
        *out = h.release();
    });
}
void oro_calib_free(void* c) { delete static_cast<CalibH*>(c); }

long oro_calib_count(void* c, int which) {
    auto& k = static_cast<CalibH*>(c)->c;
    return static_cast<long>(which == 0 ? k.scan.size() : k.lin.size());
}

int oro_calib_get(void* c, int which, std::size_t idx, double* theta, double* s_in, double* s_full,
                  std::uint8_t* excluded) {
    return guarded([&] {
        auto& k = static_cast<CalibH*>(c)->c;
        auto& v = which == 0 ? k.scan : k.lin;
        oro::require(idx < v.size(), "calib_get: index out of range");
        const oro::TCal& t = v[idx];
        if (theta) *theta = t.theta;
        if (s_in) std::memcpy(s_in, t.s_in.data(), t.s_in.size() * sizeof(double));
        if (s_full) std::memcpy(s_full, t.s_full.data(), t.s_full.size() * sizeof(double));
        if (excluded)
            for (std::size_t i = 0; i < t.excluded.size(); ++i) excluded[i] = static_cast<std::uint8_t>(t.excluded[i]);
    });
}

int oro_calib_set(void* c, int which, std::size_t idx, double theta, const double* s_in, const double* s_full,
                  const std::uint8_t* excluded) {
    return guarded([&] {
        auto& k = static_cast<CalibH*>(c)->c;
        auto& v = which == 0 ? k.scan : k.lin;
        oro::require(idx < v.size(), "calib_set: index out of range");
        oro::TCal& t = v[idx];
        t.theta = theta;
        if (s_in) std::memcpy(t.s_in.data(), s_in, t.s_in.size() * sizeof(double));
        if (s_full) std::memcpy(t.s_full.data(), s_full, t.s_full.size() * sizeof(double));
        if (excluded)
            for (std::size_t i = 0; i < t.excluded.size(); ++i) t.excluded[i] = excluded[i] ? 1 : 0;
    });
}

// mode: 0 FP (FP weights, no activation quantization: the reference's bypass),
// 1 dynamic, 2 static (quant.hpp:101).
int oro_forward(void* m, void* c, int mode, int d1, int d2, const double* images, std::size_t B, int threads,
                double* logits) {
    return guarded([&] {
        const oro::ModelW& w = static_cast<ModelH*>(m)->w;
        oro::Mode md = static_cast<oro::Mode>(mode);
        std::unique_ptr<oro::QModel> q;
        const oro::Calib* cal = nullptr;
        if (md != oro::MODE_FP) {
            oro::require(c != nullptr, "forward: quantized modes need a calibration");
            cal = &static_cast<CalibH*>(c)->c;
            q = std::make_unique<oro::QModel>(oro::quantize_model<OPS>(w, cal->spec.wbits));
        }
        oro::Driver<OPS> drv(w, q.get(), cal, md, d1 != 0, d2 != 0);
        drv.batch(images, B, logits, threads, nullptr);
    });
}

// Runs one sample and keeps every intermediate of one block (teacher-forcing
// fixtures); also the patch-embedded input and the logits.
int oro_trace(void* m, void* c, int mode, int d1, int d2, const double* image, std::size_t block, void** out) {
    return guarded([&] {
        const oro::ModelW& w = static_cast<ModelH*>(m)->w;
        oro::Mode md = static_cast<oro::Mode>(mode);
        std::unique_ptr<oro::QModel> q;
        const oro::Calib* cal = nullptr;
        if (md != oro::MODE_FP) {
            cal = &static_cast<CalibH*>(c)->c;
            q = std::make_unique<oro::QModel>(oro::quantize_model<OPS>(w, cal->spec.wbits));
        }
        oro::Driver<OPS> drv(w, q.get(), cal, md, d1 != 0, d2 != 0);
        oro::BlockTrace bt;
        std::vector<double> logits(w.d.classes), xe;
        drv.sample(image, logits.data(), block, &bt, nullptr, &xe);
        auto th = std::make_unique<TraceH>();
        put(*th, "logits", logits);
        put(*th, "x_embed", xe);
        put(*th, "x_in", bt.x_in);
        put(*th, "xn", bt.xn);
        put(*th, "u0", bt.u0);
        put(*th, "gate", bt.gate);
        put(*th, "gate_pre", bt.gpre);
        put(*th, "u", bt.u);
        put(*th, "merged", bt.merged);
        put(*th, "y", bt.y);
        put(*th, "x_out", bt.x_out);
        for (std::size_t s = 0; s < w.orders.size() + 2; ++s) {
            const oro::LinTrace& lt = bt.lin[s];
            std::string p = "lin" + std::to_string(s) + ".";
            put(*th, p + "codes", lt.codes);
            put(*th, p + "ocode", lt.ocode);
            put(*th, p + "omask", lt.omask);
            put(*th, p + "oscale", lt.oscale);
            put(*th, p + "acc_in", lt.acc_in);
            put(*th, p + "acc_out", lt.acc_out);
            put(*th, p + "out", lt.out);
            put(*th, p + "scanned", lt.scanned);
        }
        for (std::size_t d = 0; d < bt.dirs.size(); ++d) {
            const oro::DirTrace& dt = bt.dirs[d];
            std::string p = "dir" + std::to_string(d) + ".";
            put(*th, p + "u", dt.u);
            put(*th, p + "delta", dt.delta);
            put(*th, p + "bvec", dt.bvec);
            put(*th, p + "cvec", dt.cvec);
            put(*th, p + "o", dt.o);
            for (int k = 0; k < 3; ++k) {
                put(*th, p + "mask" + std::to_string(k), dt.mask[k]);
                put(*th, p + "scanned" + std::to_string(k), dt.scanned[k]);
            }
        }
        *out = th.release();
    });
}
long oro_trace_get(void* t, const char* key, void* out, std::size_t cap_bytes) {
    auto& b = static_cast<TraceH*>(t)->blobs;
    auto it = b.find(key);
    if (it == b.end()) return -1;
    if (out) std::memcpy(out, it->second.data(), std::min(cap_bytes, it->second.size()));
    return static_cast<long>(it->second.size());
}
void oro_trace_free(void* t) { delete static_cast<TraceH*>(t); }

// ---- operator-level entry points ---------------------------------------------

// The QuantHook policy (quant.cpp:467-491) over S independent streams of T
// planes of e channels x n values (plane layout x[ch*n+s], quant.cpp:313-351),
// fresh state per stream. x is fake-quantized in place; masks[S][T][e] receive
// O(t) after detection and scanned[S][T] the detect trigger.
int oro_quant_stream(double* x, std::size_t S, std::size_t T, std::size_t e, std::size_t n, double theta,
                     const double* s_in, const double* s_full, std::size_t n_refresh, unsigned abits,
                     unsigned obits, int mode, std::uint8_t* masks, std::uint8_t* scanned) {
    return guarded([&] {
        for (std::size_t s = 0; s < S; ++s) {
            typename OPS::State st;
            for (std::size_t t = 0; t < T; ++t) {
                double* p = x + (s * T + t) * e * n;
                bool sc = false;
                if (mode == oro::MODE_STATIC) {
                    OPS::fake_quant(p, e, n, nullptr, s_full[t], abits, obits);
                } else if (mode == oro::MODE_DYNAMIC) {
                    OPS::refresh(st, t, n_refresh);
                    sc = OPS::detect(st, p, e, n, theta, s_in[t], abits);
                    OPS::fake_quant(p, e, n, &st, s_in[t], abits, obits);
                    if (masks)
                        for (std::size_t ch : OPS::list(st, e)) masks[(s * T + t) * e + ch] = 1;
                }
                if (scanned) scanned[s * T + t] = sc;
            }
        }
    });
}

// hybrid_gemm (gemm.cpp:181-225) on code planes: w m x k int8 (|code|<=7),
// x_inlier k x c int8, outliers n_o channels (strictly increasing) with
// n_o x c codes and n_o scales. Outputs are m x c.
int oro_hybrid_gemm(const std::int8_t* w, const double* w_scales, std::size_t m, std::size_t k,
                    const std::int8_t* x_inlier, std::size_t c, double s_in, const std::size_t* channels,
                    std::size_t n_o, const std::int8_t* ocodes, const double* oscales, std::int32_t* acc_in,
                    std::int32_t* acc_out, double* out) {
    return guarded([&] {
        oro::OutlierBuffer ob;
        ob.cols = c;
        ob.channels.assign(channels, channels + n_o);
        ob.codes.assign(ocodes, ocodes + n_o * c);
        ob.scales.assign(oscales, oscales + n_o);
        oro::GemmResult g = OPS::hybrid_raw(w, w_scales, m, k, x_inlier, c, s_in, ob);
        if (acc_in) std::memcpy(acc_in, g.acc_inlier.data(), m * c * sizeof(std::int32_t));
        if (acc_out) std::memcpy(acc_out, g.acc_outlier.data(), m * c * sizeof(std::int32_t));
        if (out) std::memcpy(out, g.output.data(), m * c * sizeof(double));
    });
}

// split_quantize (gemm.cpp:106-135): x k x c f64 -> inlier k x c int8 and the
// outlier rows (n_o x c codes, n_o scales) of the given channel list.
int oro_split_quantize(const double* x, std::size_t k, std::size_t c, const std::size_t* channels,
                       std::size_t n_o, double s_in, unsigned abits, unsigned obits, std::int8_t* inlier,
                       std::int8_t* ocodes, double* oscales) {
    return guarded([&] {
        std::vector<std::size_t> ol(channels, channels + n_o);
        oro::SplitOperands sp = OPS::split(x, k, c, ol, s_in, abits, obits);
        std::memcpy(inlier, sp.inlier_codes.data(), k * c);
        if (n_o) {
            std::memcpy(ocodes, sp.outliers.codes.data(), n_o * c);
            std::memcpy(oscales, sp.outliers.scales.data(), n_o * sizeof(double));
        }
    });
}

// pack_int4 (gemm.cpp:60-76).
int oro_pack_int4(const std::int8_t* codes, std::size_t rows, std::size_t cols, std::uint8_t* out) {
    return guarded([&] {
        auto b = OPS::pack(codes, rows, cols);
        std::memcpy(out, b.data(), b.size());
    });
}

}  // extern "C"
