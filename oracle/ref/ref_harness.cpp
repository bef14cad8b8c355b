// ORACLE (reference build) — test infrastructure only.
//
// _ref/libouro_ref.so: the shared model driver (oracle/driver.hpp) running on
// the reference's OWN compiled primitives (sources compiled in place from
// /root/reference/proj/src/ouro, never copied): make_toy_model, quantize_weights,
// detail::mm, softplus_val/silu_val, maybe_refresh, detect_outliers,
// fake_quant_step, split_quantize, pack_int4, hybrid_gemm. Plus pin entry points
// that call the reference's exported end-to-end functions (vmm_forward_raw,
// quantized_forward, calibrate) so the driver's restatement of the reference's
// anonymous-namespace code (block, QuantHook, recorder) is checked bit-for-bit.
#include <cstring>

#include "../oracle_ops.hpp"
#include "ouro/config.hpp"
#include "ouro/gemm.hpp"
#include "ouro/pipeline.hpp"
#include "ouro/tensor_io.hpp"
#include "ouro/quant.hpp"
#include "ouro/ssm.hpp"
#include "ouro/tensor.hpp"

namespace oro {

inline std::vector<double> tvec(const ouro::Tensor& t) { return std::vector<double>(t.ptr(), t.ptr() + t.numel()); }
inline void tset(ouro::Tensor& t, const std::vector<double>& v) { std::memcpy(t.mut(), v.data(), v.size() * sizeof(double)); }

inline ouro::ModelDims to_ref(const Dims& d) {
    ouro::ModelDims r;
    r.image = d.image;
    r.channels = d.channels;
    r.patch = d.patch;
    r.embed = d.embed;
    r.state = d.state;
    r.blocks = d.blocks;
    r.classes = d.classes;
    r.conv_width = d.conv_width;
    return r;
}

inline ouro::ToyVmmModel to_ref(const ModelW& w) {
    std::vector<ouro::ScanOrder> ord;
    for (int o : w.orders) ord.push_back(static_cast<ouro::ScanOrder>(o));
    ouro::ToyVmmModel m = ouro::make_toy_model(to_ref(w.d), ord, 0);
    tset(m.patch_embed_w, w.patch_w);
    tset(m.patch_embed_b, w.patch_b);
    tset(m.head_w, w.head_w);
    tset(m.head_b, w.head_b);
    for (std::size_t b = 0; b < w.blocks.size(); ++b) {
        tset(m.blocks[b].w_in, w.blocks[b].w_in);
        tset(m.blocks[b].w_gate, w.blocks[b].w_gate);
        tset(m.blocks[b].conv, w.blocks[b].conv);
        tset(m.blocks[b].out_proj, w.blocks[b].out_proj);
        for (std::size_t d = 0; d < w.blocks[b].dirs.size(); ++d) {
            auto& p = m.blocks[b].dirs[d];
            const auto& q = w.blocks[b].dirs[d];
            tset(p.a, q.a);
            tset(p.w_b, q.w_b);
            tset(p.w_c, q.w_c);
            tset(p.w_delta, q.w_delta);
            tset(p.b_delta, q.b_delta);
        }
    }
    return m;
}

struct RefOps {
    using State = ouro::OutlierState;
    struct Weight {
        ouro::PackedInt4 packed;
        std::vector<std::int8_t> codes;
        std::vector<double> scales;
        std::size_t rows = 0, cols = 0;
    };
    struct Prepared;

    static ModelW make_model(const Dims& d, const std::vector<int>& orders, std::uint64_t seed) {
        std::vector<ouro::ScanOrder> ord;
        for (int o : orders) ord.push_back(static_cast<ouro::ScanOrder>(o));
        ouro::ToyVmmModel m = ouro::make_toy_model(to_ref(d), ord, seed);
        ModelW w;
        w.d = d;
        w.orders = orders;
        w.patch_w = tvec(m.patch_embed_w);
        w.patch_b = tvec(m.patch_embed_b);
        w.head_w = tvec(m.head_w);
        w.head_b = tvec(m.head_b);
        for (auto& b : m.blocks) {
            BlockW bw;
            bw.w_in = tvec(b.w_in);
            bw.w_gate = tvec(b.w_gate);
            bw.conv = tvec(b.conv);
            bw.out_proj = tvec(b.out_proj);
            for (auto& p : b.dirs) {
                DirW dw;
                dw.a = tvec(p.a);
                dw.w_b = tvec(p.w_b);
                dw.w_c = tvec(p.w_c);
                dw.w_delta = tvec(p.w_delta);
                dw.b_delta = tvec(p.b_delta);
                bw.dirs.push_back(std::move(dw));
            }
            w.blocks.push_back(std::move(bw));
        }
        return w;
    }
    static QRows quantize_rows(const std::vector<double>& w, std::size_t rows, unsigned bits) {
        ouro::Tensor t = ouro::Tensor::zeros({rows, w.size() / rows});
        tset(t, w);
        ouro::QuantizedRows q = ouro::quantize_weights(t, bits);
        QRows r;
        r.codes = q.codes;
        r.scales = q.scales;
        r.deq = tvec(ouro::dequantize_rows(q));
        return r;
    }
    static void mm_nt(const double* a, const double* b, double* c, std::size_t m, std::size_t k, std::size_t n) {
        ouro::detail::mm(a, b, c, m, k, n, false, true, false);
    }
    static double softplus(double x) { return ouro::detail::softplus_val(x); }
    static double silu(double x) { return ouro::detail::silu_val(x); }
    static void refresh(State& st, std::size_t t, std::size_t n) { ouro::maybe_refresh(st, t, n); }
    static bool detect(State& st, const double* x, std::size_t e, std::size_t n, double th, double s, unsigned b) {
        return ouro::detect_outliers(st, x, e, n, th, s, b).scanned;
    }
    static void fake_quant(double* x, std::size_t e, std::size_t n, const State* st, double s, unsigned ab,
                           unsigned ob) {
        ouro::OutlierState none;
        ouro::fake_quant_step(x, e, n, st ? *st : none, s, ab, ob);
    }
    static std::vector<std::size_t> list(const State& st, std::size_t) { return st.o_list; }
    static SplitOperands split(const double* x, std::size_t k, std::size_t c, const std::vector<std::size_t>& o,
                               double s, unsigned ab, unsigned ob) {
        ouro::SplitOperands r = ouro::split_quantize(x, k, c, o, s, ab, ob);
        SplitOperands out;
        out.inlier_codes = r.inlier_codes;
        out.outliers.channels = r.outliers.channels;
        out.outliers.codes = r.outliers.codes;
        out.outliers.scales = r.outliers.scales;
        out.outliers.cols = r.outliers.cols;
        return out;
    }
    static GemmResult run_hybrid(const ouro::PackedInt4* wp, const std::int8_t* w, const double* ws, std::size_t m,
                                 std::size_t k, const std::int8_t* x, std::size_t c, double s,
                                 const OutlierBuffer& ob) {
        bool a4 = true;
        for (std::size_t i = 0; i < k * c; ++i) a4 = a4 && x[i] >= -7 && x[i] <= 7;
        if (!a4)  // A8 inliers cannot be packed (gemm.cpp:69); the reference's own A8
                  // oracle is the triple loop (tests/test_gemm.cpp:25-35) -> restated form.
            return hybrid_gemm(w, ws, m, k, x, c, s, ob);
        ouro::PackedInt4 local;
        if (!wp) {
            local = ouro::pack_int4(w, m, k);
            wp = &local;
        }
        ouro::OutlierBuffer rb;
        rb.channels = ob.channels;
        rb.codes = ob.codes;
        rb.scales = ob.scales;
        rb.cols = c;
        ouro::GemmResult g = ouro::hybrid_gemm(*wp, std::vector<double>(ws, ws + m), ouro::pack_int4(x, k, c), s, rb, 1,
                                               false);
        GemmResult r;
        r.acc_inlier = g.acc_inlier;
        r.acc_outlier = g.acc_outlier;
        r.output = g.output;
        return r;
    }
    static GemmResult hybrid(const Weight& w, const SplitOperands& sp, double s) {
        return run_hybrid(&w.packed, w.codes.data(), w.scales.data(), w.rows, w.cols, sp.inlier_codes.data(), 1, s,
                          sp.outliers);
    }
    static GemmResult hybrid_raw(const std::int8_t* w, const double* ws, std::size_t m, std::size_t k,
                                 const std::int8_t* x, std::size_t c, double s, const OutlierBuffer& ob) {
        return run_hybrid(nullptr, w, ws, m, k, x, c, s, ob);
    }
    static std::vector<std::uint8_t> pack(const std::int8_t* codes, std::size_t r, std::size_t c) {
        return ouro::pack_int4(codes, r, c).bytes;
    }
    template <class Q>
    static Prepared prepare(const Q& q);
};

}  // namespace oro

#include "../driver.hpp"

namespace oro {
struct RefOps::Prepared {
    struct Blk {
        Weight in, out;
        std::vector<Weight> xp;
    };
    std::vector<Blk> blocks;
};
template <class Q>
RefOps::Prepared RefOps::prepare(const Q& q) {
    auto mk = [](const QRows& r) {
        Weight w;
        w.codes = r.codes;
        w.scales = r.scales;
        w.rows = r.scales.size();
        w.cols = r.codes.size() / w.rows;
        w.packed = ouro::pack_int4(w.codes.data(), w.rows, w.cols);
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

using OPS = oro::RefOps;
#include "../capi_impl.hpp"

// ---- pins: the reference's exported end-to-end functions ----------------------
extern "C" {

// vmm_forward_raw (ssm.cpp:237-277) with no hook: FP logits, no D1/D2.
int ref_pin_fp_forward(void* m, const double* images, std::size_t B, double* logits) {
    return guarded([&] {
        const oro::ModelW& w = static_cast<ModelH*>(m)->w;
        ouro::ToyVmmModel rm = oro::to_ref(w);
        std::size_t pix = w.d.image * w.d.image * w.d.channels;
        ouro::RawForward r = ouro::vmm_forward_raw(rm, std::vector<double>(images, images + B * pix), B, nullptr, false);
        std::memcpy(logits, r.logits.data(), r.logits.size() * sizeof(double));
    });
}

// calibrate (quant.cpp:129-177) into a calib handle (scan tensors only).
int ref_pin_calibrate(void* m, const double* images, std::size_t B, const unsigned* bits, std::size_t n_refresh,
                      double rho, void** out) {
    return guarded([&] {
        const oro::ModelW& w = static_cast<ModelH*>(m)->w;
        ouro::ToyVmmModel rm = oro::to_ref(w);
        std::size_t pix = w.d.image * w.d.image * w.d.channels;
        ouro::QuantSpec spec;
        spec.weight_bits = bits[0];
        spec.act_bits = bits[1];
        spec.outlier_bits = bits[2];
        spec.n_refresh = n_refresh;
        spec.rho = rho;
        ouro::CalibrationResult cr = ouro::calibrate(rm, std::vector<double>(images, images + B * pix), B, spec);
        auto h = std::make_unique<CalibH>();
        oro::Calib& c = h->c;
        c.spec = make_spec(bits, n_refresh, rho);
        c.tokens = cr.tokens;
        c.embed = cr.embed;
        c.state = cr.state;
        c.blocks = cr.blocks;
        c.ndirs = cr.ndirs;
        c.d1 = false;
        c.d2 = false;
        for (const auto& t : cr.tensors) {
            oro::TCal tc;
            tc.theta = t.theta;
            tc.s_in = t.scale_inlier;
            tc.s_full = t.scale_full;
            tc.excluded = t.excluded;
            c.scan.push_back(std::move(tc));
        }
        *out = h.release();
    });
}

// quantized_forward (quant.cpp:505-579): logits of the quantized pass
// (mode 1 dynamic / 2 static / 3 bypass) under a calibration handle.
int ref_pin_quantized_forward(void* m, void* c, int mode, const double* images, std::size_t B, double* logits_q,
                              double* logits_fp) {
    return guarded([&] {
        const oro::ModelW& w = static_cast<ModelH*>(m)->w;
        const oro::Calib& k = static_cast<CalibH*>(c)->c;
        ouro::ToyVmmModel rm = oro::to_ref(w);
        std::size_t pix = w.d.image * w.d.image * w.d.channels;
        ouro::CalibrationResult cr;
        cr.spec.weight_bits = k.spec.wbits;
        cr.spec.act_bits = k.spec.abits;
        cr.spec.outlier_bits = k.spec.obits;
        cr.spec.n_refresh = k.spec.n_refresh;
        cr.spec.rho = k.spec.rho;
        cr.tokens = k.tokens;
        cr.embed = k.embed;
        cr.state = k.state;
        cr.blocks = k.blocks;
        cr.ndirs = k.ndirs;
        for (const auto& t : k.scan) {
            ouro::TensorCalib tc;
            tc.theta = t.theta;
            tc.scale_inlier = t.s_in;
            tc.scale_full = t.s_full;
            tc.excluded = t.excluded;
            cr.tensors.push_back(std::move(tc));
        }
        ouro::QuantMode qm = mode == 1 ? ouro::QuantMode::Dynamic
                                       : (mode == 2 ? ouro::QuantMode::Static : ouro::QuantMode::Bypass);
        ouro::QuantEvalResult r = ouro::quantized_forward(rm, std::vector<double>(images, images + B * pix), B, cr, qm,
                                                          ouro::SpikeSettings{});
        std::memcpy(logits_q, r.logits_q.data(), r.logits_q.size() * sizeof(double));
        if (logits_fp) std::memcpy(logits_fp, r.logits_fp.data(), r.logits_fp.size() * sizeof(double));
    });
}

// quantized_forward (quant.cpp:505-579) with its metrics: logits_mse, argmax
// agreement and the teacher-forced per-(block, dir) scan MSE (no spikes).
static void quant_eval_impl(void* m, void* c, int mode, const double* images, std::size_t B, double* logits_q,
                            double* logits_fp, double* logits_mse, std::size_t* argmax_agree, double* layer_mse,
                            const ouro::SpikeSettings& spikes) {
    {
        const oro::ModelW& w = static_cast<ModelH*>(m)->w;
        const oro::Calib& k = static_cast<CalibH*>(c)->c;
        ouro::ToyVmmModel rm = oro::to_ref(w);
        std::size_t pix = w.d.image * w.d.image * w.d.channels;
        ouro::CalibrationResult cr;
        cr.spec.weight_bits = k.spec.wbits;
        cr.spec.act_bits = k.spec.abits;
        cr.spec.outlier_bits = k.spec.obits;
        cr.spec.n_refresh = k.spec.n_refresh;
        cr.spec.rho = k.spec.rho;
        cr.tokens = k.tokens;
        cr.embed = k.embed;
        cr.state = k.state;
        cr.blocks = k.blocks;
        cr.ndirs = k.ndirs;
        for (const oro::TCal& t : k.scan) {
            ouro::TensorCalib tc;
            tc.theta = t.theta;
            tc.scale_inlier = t.s_in;
            tc.scale_full = t.s_full;
            tc.excluded.assign(t.excluded.begin(), t.excluded.end());
            cr.tensors.push_back(std::move(tc));
        }
        ouro::QuantMode qm = mode == 1 ? ouro::QuantMode::Dynamic
                                       : (mode == 2 ? ouro::QuantMode::Static : ouro::QuantMode::Bypass);
        ouro::QuantEvalResult r = ouro::quantized_forward(rm, std::vector<double>(images, images + B * pix), B, cr, qm,
                                                          spikes);
        std::memcpy(logits_q, r.logits_q.data(), r.logits_q.size() * sizeof(double));
        std::memcpy(logits_fp, r.logits_fp.data(), r.logits_fp.size() * sizeof(double));
        *logits_mse = r.logits_mse;
        *argmax_agree = r.argmax_agree;
        for (std::size_t i = 0; i < r.layer_mse.size(); ++i) layer_mse[i] = r.layer_mse[i].second;
    }
}

int ref_pin_quant_eval(void* m, void* c, int mode, const double* images, std::size_t B, double* logits_q,
                       double* logits_fp, double* logits_mse, std::size_t* argmax_agree, double* layer_mse) {
    return guarded([&] {
        quant_eval_impl(m, c, mode, images, B, logits_q, logits_fp, logits_mse, argmax_agree, layer_mse,
                        ouro::SpikeSettings{});
    });
}

// quantized_forward with SpikeSettings (quant.hpp:105-110, SpikeHook quant.cpp:420-446).
int ref_pin_quant_eval_spiked(void* m, void* c, int mode, const double* images, std::size_t B, double* logits_q,
                              double* logits_fp, double* logits_mse, std::size_t* argmax_agree, double* layer_mse,
                              double rate, double gain, std::size_t channels, std::uint64_t salt) {
    return guarded([&] {
        ouro::SpikeSettings sp;
        sp.rate = rate;
        sp.gain = gain;
        sp.channels = channels;
        sp.salt = salt;
        quant_eval_impl(m, c, mode, images, B, logits_q, logits_fp, logits_mse, argmax_agree, layer_mse, sp);
    });
}

// bench_refresh_sweep (gemm.cpp:326-411) itself: per period, the mean |O| after
// detection and the scans per step (the GPU sweep draws the same operands).
int ref_pin_refresh_sweep(const std::size_t* periods, std::size_t n_periods, std::size_t steps, std::size_t m,
                          std::size_t k, std::size_t c, std::size_t persistent, double transient_rate,
                          double spike_gain, std::size_t trials, std::uint64_t seed, double* mean_o_list,
                          double* scans_per_step) {
    return guarded([&] {
        ouro::SweepSettings ss;
        ss.periods.assign(periods, periods + n_periods);
        ss.steps = steps;
        ss.m = m;
        ss.k = k;
        ss.c = c;
        ss.persistent_channels = persistent;
        ss.transient_rate = transient_rate;
        ss.spike_gain = spike_gain;
        ss.trials = trials;
        ss.seed = seed;
        const auto recs = ouro::bench_refresh_sweep(ss);
        for (std::size_t i = 0; i < recs.size(); ++i) {
            mean_o_list[i] = recs[i].mean_o_list;
            scans_per_step[i] = recs[i].scans_per_step;
        }
    });
}

// bench_gemm (gemm.cpp:260-324): the record list (path 0 hybrid / 1 f64, size).
int ref_pin_gemm_bench(const std::size_t* sizes, std::size_t n_sizes, double outlier_fraction, std::size_t trials,
                       std::uint64_t seed, int* paths, std::size_t* out_sizes) {
    return guarded([&] {
        ouro::BenchSettings bs;
        bs.sizes.assign(sizes, sizes + n_sizes);
        bs.outlier_fraction = outlier_fraction;
        bs.trials = trials;
        bs.seed = seed;
        const auto recs = ouro::bench_gemm(bs);
        for (std::size_t i = 0; i < recs.size(); ++i) {
            paths[i] = recs[i].path == "hybrid" ? 0 : 1;
            out_sizes[i] = recs[i].size;
        }
    });
}

// save_calibration (quant.cpp:179-216) of a calibration handle's scan tensors,
// named block<b>.dir<d>.<kind> as calibrate names them (quant.cpp:150-151).
int ref_pin_save_calibration(void* c, const char* dir) {
    return guarded([&] {
        const oro::Calib& k = static_cast<CalibH*>(c)->c;
        ouro::CalibrationResult cr;
        cr.spec.weight_bits = k.spec.wbits;
        cr.spec.act_bits = k.spec.abits;
        cr.spec.outlier_bits = k.spec.obits;
        cr.spec.n_refresh = k.spec.n_refresh;
        cr.spec.rho = k.spec.rho;
        cr.tokens = k.tokens;
        cr.embed = k.embed;
        cr.state = k.state;
        cr.blocks = k.blocks;
        cr.ndirs = k.ndirs;
        const char* kinds[3] = {"a_bar", "b_bar", "h"};
        for (std::size_t b = 0; b < k.blocks; ++b)
            for (std::size_t d = 0; d < k.ndirs; ++d)
                for (int q = 0; q < 3; ++q) {
                    const oro::TCal& t = k.at(b, d, q);
                    ouro::TensorCalib tc;
                    tc.name = "block" + std::to_string(b) + ".dir" + std::to_string(d) + "." + kinds[q];
                    tc.theta = t.theta;
                    tc.scale_inlier = t.s_in;
                    tc.scale_full = t.s_full;
                    tc.excluded.assign(t.excluded.begin(), t.excluded.end());
                    cr.tensors.push_back(std::move(tc));
                }
        ouro::save_calibration(dir, cr);
    });
}

// load_calibration (quant.cpp:218-290) into a calibration handle (scan tensors).
int ref_pin_load_calibration(const char* dir, void** out) {
    return guarded([&] {
        ouro::CalibrationResult cr = ouro::load_calibration(dir);
        auto h = std::make_unique<CalibH>();
        oro::Calib& c = h->c;
        const unsigned bits[3] = {cr.spec.weight_bits, cr.spec.act_bits, cr.spec.outlier_bits};
        c.spec = make_spec(bits, cr.spec.n_refresh, cr.spec.rho);
        c.tokens = cr.tokens;
        c.embed = cr.embed;
        c.state = cr.state;
        c.blocks = cr.blocks;
        c.ndirs = cr.ndirs;
        c.d1 = false;
        c.d2 = false;
        for (const auto& t : cr.tensors) {
            oro::TCal tc;
            tc.theta = t.theta;
            tc.s_in = t.scale_inlier;
            tc.s_full = t.scale_full;
            tc.excluded = t.excluded;
            c.scan.push_back(std::move(tc));
        }
        *out = h.release();
    });
}

// The reference's own pipeline stages (pipeline.cpp), driven by a config text in
// the reference's format (parse_config_text): the stage entry points of the B200
// C ABI (ouro_b200_quant_eval / ouro_b200_calib_stage) are checked against these
// file for file. run_id_of gives the metrics lines' run tag.
int ref_pin_run_id(const char* config_text, char* out, std::size_t cap) {
    return guarded([&] {
        const std::string id = ouro::run_id_of(ouro::parse_config_text(config_text));
        if (id.size() + 1 > cap) throw ouro::ValidationError("run id buffer too small");
        std::memcpy(out, id.c_str(), id.size() + 1);
    });
}
int ref_pin_run_quant_eval(const char* config_text, const char* calib_dir, const char* images_file,
                           const char* out_dir) {
    return guarded([&] { ouro::run_quant_eval(ouro::parse_config_text(config_text), calib_dir, images_file, out_dir); });
}
int ref_pin_run_calib(const char* config_text, const char* images_file, const char* out_dir) {
    return guarded([&] { ouro::run_calib(ouro::parse_config_text(config_text), images_file, out_dir); });
}
// write_tensor_f64 / _i8 / _u4 and their readers (tensor_io.cpp), for the
// OURO container parity tests
int ref_pin_write_tensor(const char* path, int dtype, const std::uint64_t* shape, std::size_t rank, const void* data) {
    return guarded([&] {
        ouro::Shape sh(shape, shape + rank);
        std::size_t n = 1;
        for (std::size_t d : sh) n *= d;
        if (dtype == 0) {
            ouro::write_tensor_f64(path, ouro::Tensor::from(sh, std::vector<double>(static_cast<const double*>(data),
                                                                                    static_cast<const double*>(data) + n)));
        } else {
            std::vector<std::int8_t> v(static_cast<const std::int8_t*>(data), static_cast<const std::int8_t*>(data) + n);
            if (dtype == 1) ouro::write_tensor_i8(path, sh, v);
            else ouro::write_tensor_u4(path, sh, v);
        }
    });
}
int ref_pin_read_tensor_codes(const char* path, int dtype, std::int8_t* out, std::size_t cap, std::size_t* n) {
    return guarded([&] {
        auto r = dtype == 1 ? ouro::read_tensor_i8(path) : ouro::read_tensor_u4(path);
        *n = r.second.size();
        if (r.second.size() > cap) throw ouro::ValidationError("output buffer too small");
        std::memcpy(out, r.second.data(), r.second.size());
    });
}

}  // extern "C"
