// Pipeline stage entry points and OURO tensor files at the C ABI (SURVEY §8(f)
// 3-4): the GPU-backed forms of the reference's ouro_quant_eval / ouro_calib
// (ouromamba.h:58-65, capi.cpp:166-186) and of write_tensor_* / read_tensor_*
// (tensor_io.hpp:21-31).
//
// quant-eval (run_quant_eval, pipeline.cpp:115-167): model from the config's
// dims + seed (make_toy_model), calibration directory, image batch file (OURO
// f64 [B, H*W*C]), eval_batch images; quantized_forward's metrics (quant.cpp:
// 505-579) computed on the GPU — FP and quantized logits, logits_mse, argmax
// agreement, the teacher-forced scan-output MSE per (block, dir) (each direction's
// quantized scan re-run on the FP pass's own scan input with the W4 x_proj
// weights), and the QuantHook timeline (sample 0, b_bar tensors: |O| after
// maybe_refresh and after detect_outliers per step, quant.cpp:485-487) — written
// as metrics.txt in the reference's line format (format_metrics_line,
// config.cpp:409-420, "%.17g" doubles), plus a manifest.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>

#include "../../include/ouro_b200.h"
#include "engine.h"
#include "common.cuh"
#include "guard.h"

namespace ob {
namespace {

std::string g17(double v) {  // fmt_double, config.cpp:259-263
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

using KV = std::vector<std::pair<std::string, std::string>>;
std::string metrics_line(const std::string& run, const std::string& stage, const KV& kv) {  // config.cpp:409-420
    std::string out = "run=" + run + " stage=" + stage;
    for (const auto& [k, v] : kv) {
        require(k.find_first_of(" =\n") == std::string::npos && v.find_first_of(" \n") == std::string::npos,
                "metrics: keys and values must not contain spaces or newlines");
        out += " " + k + "=" + v;
    }
    return out + "\n";
}

Dims dims_of(const ouro_b200_stage_config& c) {
    Dims d;
    d.image = static_cast<int>(c.image);
    d.channels = static_cast<int>(c.channels);
    d.patch = static_cast<int>(c.patch);
    d.embed = static_cast<int>(c.embed);
    d.state = static_cast<int>(c.state);
    d.blocks = static_cast<int>(c.blocks);
    d.classes = static_cast<int>(c.classes);
    d.conv_width = static_cast<int>(c.conv_width);
    return d;
}

QuantSpec spec_of(const ouro_b200_stage_config& c) {  // quant_spec_from_config, pipeline.cpp:27-36
    QuantSpec s;
    s.wbits = c.weight_bits;
    s.abits = c.act_bits;
    s.obits = c.outlier_bits;
    s.n_refresh = static_cast<int>(c.n_refresh);
    s.rho = c.outlier_quantile;
    s.validate();
    require(s.abits <= 8 && s.wbits <= 4, "stage config: bit widths outside this build's operands");
    return s;
}

int mode_of(const char* name) {  // quant_mode_from_name
    require(name != nullptr, "stage config: quant mode is NULL");
    const std::string m(name);
    if (m == "dynamic") return MODE_DYNAMIC;
    if (m == "static") return MODE_STATIC;
    if (m == "bypass") return MODE_FP;
    throw ValidationError("config: quant.mode must be dynamic, static or bypass, got '" + m + "'");
}

// Image batch file: rank-2, rows = samples, cols = flattened pixels (pipeline.cpp:39-49).
std::vector<double> load_images(const std::string& file, size_t pix, size_t* batch) {
    const OuroTensor t = ouro_tensor_read(file);
    if (t.dtype != OuroDtype::F64) throw IoError(file + ": dtype mismatch, file holds tag " +
                                                 std::to_string(static_cast<unsigned>(t.dtype)));
    std::string shape = "[";
    for (size_t i = 0; i < t.shape.size(); ++i) shape += (i ? "," : "") + std::to_string(t.shape[i]);
    shape += "]";
    require(t.shape.size() == 2 && t.shape[1] == pix && t.shape[0] >= 1,
            "image batch " + file + ": expected shape [B," + std::to_string(pix) + "], got " + shape);
    *batch = static_cast<size_t>(t.shape[0]);
    const double* p = reinterpret_cast<const double*>(t.payload.data());
    return std::vector<double>(p, p + *batch * pix);
}

void ensure_dir(const std::string& dir) {
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    if (ec) throw IoError("cannot create directory " + dir + ": " + ec.message());
}

std::string manifest(const ouro_b200_stage_config& c, const std::string& run, const std::string& stage,
                     const KV& extra) {
    std::string o = "[model]\n";
    o += "seed = " + std::to_string(c.seed) + "\nimage = " + std::to_string(c.image) +
         "\nchannels = " + std::to_string(c.channels) + "\npatch = " + std::to_string(c.patch) +
         "\nembed = " + std::to_string(c.embed) + "\nstate = " + std::to_string(c.state) +
         "\nblocks = " + std::to_string(c.blocks) + "\nclasses = " + std::to_string(c.classes) +
         "\nconv_width = " + std::to_string(c.conv_width) + "\nscan_orders = row-forward,row-backward\n";
    o += "\n[quant]\nweight_bits = " + std::to_string(c.weight_bits) + "\nact_bits = " + std::to_string(c.act_bits) +
         "\noutlier_bits = " + std::to_string(c.outlier_bits) + "\nn_refresh = " +
         (c.n_refresh == 0 ? std::string("full") : std::to_string(c.n_refresh)) +
         "\noutlier_quantile = " + g17(c.outlier_quantile) + "\nspike_rate = " + g17(c.spike_rate) +
         "\nspike_gain = " + g17(c.spike_gain) + "\nspike_channels = " + std::to_string(c.spike_channels) +
         "\neval_batch = " + std::to_string(c.eval_batch) + "\nmode = " + std::string(c.mode ? c.mode : "") + "\n";
    o += "\n[b200]\nd1 = " + std::to_string(c.d1 ? 1 : 0) + "\nd2 = " + std::to_string(c.d2 ? 1 : 0) +
         "\ndevice = " + std::to_string(c.device) + "\n";
    o += "\n[run]\nrun_id = " + run + "\nstage = " + stage + "\nseed_source = config\n";
    for (const auto& [k, v] : extra) o += k + " = " + v + "\n";
    return o;
}

template <class T>
std::vector<T> to_host(const T* dev, size_t n, cudaStream_t st) {
    std::vector<T> h(n);
    cuda_check(cudaStreamSynchronize(st), "stage sync");
    cuda_check(cudaMemcpy(h.data(), dev, n * sizeof(T), cudaMemcpyDeviceToHost), "stage copy");
    return h;
}

template <class T>
const T* blob(const Model::TraceSink& tr, const std::string& key, size_t n) {
    auto it = tr.blobs.find(key);
    require(it != tr.blobs.end() && it->second.size() == n * sizeof(T), "internal error: trace entry " + key);
    return reinterpret_cast<const T*>(it->second.data());
}

struct EvalOut {
    std::vector<double> logits_fp, logits_q;
    double logits_mse = 0.0;
    size_t argmax_agree = 0;
    KV layer_mse;
    struct TL {
        std::string tensor;
        int t;
        int after_refresh, after_detect;
    };
    std::vector<TL> timeline;
};

// quantized_forward (quant.cpp:505-579) on the GPU.
EvalOut quant_eval(Model& m, Calibration& cal, int mode, bool d1, bool d2, const std::vector<double>& images,
                   int B, const SpikeCfg& spikes) {
    cudaStream_t st = m.ctx->stream;
    const Dims& d = m.d;
    const int L = d.tokens(), E = d.embed, N = d.state, nd = static_cast<int>(m.host.orders.size());
    const size_t pix = static_cast<size_t>(d.image) * d.image * d.channels;
    DevBuf<double> img, lg;
    img.upload(images.data(), static_cast<size_t>(B) * pix, st);
    lg.ensure(static_cast<size_t>(B) * d.classes);
    m.spikes = spikes;
    EvalOut out;
    // SpikeHook in every pass; QuantHook in the quantized one (weights W4 unless bypass)
    m.forward(&cal, mode, d1, d2, img.p, B, lg.p, nullptr, nullptr);
    out.logits_q = to_host(lg.p, static_cast<size_t>(B) * d.classes, st);
    m.forward(nullptr, MODE_FP, d1, d2, img.p, B, lg.p, nullptr, nullptr);
    out.logits_fp = to_host(lg.p, static_cast<size_t>(B) * d.classes, st);
    double lm = 0.0;
    for (size_t i = 0; i < out.logits_fp.size(); ++i) {
        const double e = out.logits_fp[i] - out.logits_q[i];
        lm += e * e;
    }
    out.logits_mse = lm / static_cast<double>(out.logits_fp.size());
    for (int b = 0; b < B; ++b) {  // std::max_element: first maximum
        const double* f = out.logits_fp.data() + static_cast<size_t>(b) * d.classes;
        const double* q = out.logits_q.data() + static_cast<size_t>(b) * d.classes;
        if (std::max_element(f, f + d.classes) - f == std::max_element(q, q + d.classes) - q) ++out.argmax_agree;
    }
    // teacher-forced per-(block, dir) scan MSE: the quantized scan re-run on the FP
    // pass's own scan input (quant.cpp:548-577); bypass re-scans the unquantized model
    const int P = E + 2 * N;
    const size_t rows = static_cast<size_t>(B) * L;
    DevBuf<double> uperm, u, proj, o_tf, w;
    u.ensure(rows * E);
    uperm.ensure(rows * E);
    proj.ensure(rows * P);
    o_tf.ensure(rows * E);
    std::vector<double> up(rows * E);
    for (int blk = 0; blk < d.blocks; ++blk) {
        Model::TraceSink tr;
        tr.block = blk;
        m.forward(nullptr, MODE_FP, d1, d2, img.p, B, lg.p, &tr, nullptr);
        const double* uh = blob<double>(tr, "u", rows * E);
        u.upload(uh, rows * E, st);
        for (int k = 0; k < nd; ++k) {
            const int order = m.host.orders[static_cast<size_t>(k)];
            for (int s = 0; s < B; ++s)
                for (int t = 0; t < L; ++t)
                    std::memcpy(up.data() + (static_cast<size_t>(s) * L + t) * E,
                                uh + (static_cast<size_t>(s) * L + row_at(order, t, L, d.grid())) * E,
                                static_cast<size_t>(E) * sizeof(double));
            uperm.upload(up.data(), rows * E, st);
            const std::string pd = "block" + std::to_string(blk) + ".dir" + std::to_string(k) + ".";
            std::vector<double> wx;
            if (mode == MODE_FP) {
                for (const char* n : {"w_delta", "w_b", "w_c"}) {
                    const auto& v = m.host.t.at(pd + n);
                    wx.insert(wx.end(), v.begin(), v.end());
                }
            } else {
                wx = m.host.dequantized(pd + "xp", cal.spec.wbits);
            }
            w.upload(wx.data(), wx.size(), st);
            DGemmParams g;  // k-ascending dots, as s6_scan's projections (tensor.cpp:373-382)
            g.M = static_cast<int>(rows);
            g.R = P;
            g.K = E;
            g.a = uperm.p;
            g.lda = E;
            g.w = w.p;
            g.epi.out = proj.p;
            g.epi.ld_out = P;
            cuda_check(launch_dgemm(g, st), "teacher-forced projection");
            ScanParams sp;
            sp.S = B;
            sp.T = L;
            sp.E = E;
            sp.N = N;
            sp.order = order;
            sp.grid = d.grid();
            sp.u = u.p;
            sp.proj = proj.p;
            sp.a = m.blocks[static_cast<size_t>(blk)].dirs[static_cast<size_t>(k)].a.p;
            sp.b_delta = m.blocks[static_cast<size_t>(blk)].dirs[static_cast<size_t>(k)].b_delta.p;
            sp.o = o_tf.p;
            sp.mode = mode;
            if (mode != MODE_FP) {
                sp.n_refresh = cal.spec.n_refresh;
                sp.abits = cal.spec.abits;
                sp.obits = cal.spec.obits;
                for (int q = 0; q < 3; ++q) {
                    const size_t si = (static_cast<size_t>(blk) * nd + k) * 3 + q;
                    sp.cal[q].theta = cal.scan[si].theta;
                    sp.cal[q].s_in = cal.s_in_dev(false, si);
                    sp.cal[q].s_full = cal.s_full_dev(false, si);
                    sp.cal[q].inv_in = cal.inv_in_dev(false, si);
                    sp.cal[q].inv_full = cal.inv_full_dev(false, si);
                }
                sp.literal = cal.literal.p + (static_cast<size_t>(blk) * nd + k) * L;
                sp.literal_any = mode == MODE_DYNAMIC ? cal.literal_any[static_cast<size_t>(blk) * nd + k] : 0;
            }
            sp.spike = spikes;
            sp.spike.block = blk;
            sp.spike.dir = k;
            cuda_check(launch_scan(sp, st, nullptr), "teacher-forced scan");
            const std::vector<double> oh = to_host(o_tf.p, rows * E, st);
            const double* of = blob<double>(tr, "dir" + std::to_string(k) + ".o", rows * E);
            // summed in the reference's order: per sample, scan step t, channel
            // (s6_scan returns o in scan order, quant.cpp:566-570); o is stored here at
            // canonical rows
            double acc = 0.0;
            for (int s = 0; s < B; ++s)
                for (int t = 0; t < L; ++t) {
                    const size_t r = (static_cast<size_t>(s) * L + row_at(order, t, L, d.grid())) * E;
                    for (int e = 0; e < E; ++e) {
                        const double df = of[r + e] - oh[r + e];
                        acc += df * df;
                    }
                }
            out.layer_mse.emplace_back("block" + std::to_string(blk) + ".dir" + std::to_string(k),
                                       g17(acc / static_cast<double>(rows * E)));
        }
    }
    // QuantHook timeline: sample 0, b_bar tensors, |O| after refresh / after detection
    if (mode == MODE_DYNAMIC) {
        for (int blk = 0; blk < d.blocks; ++blk) {
            Model::TraceSink tr;
            tr.block = blk;
            m.forward(&cal, mode, d1, d2, img.p, 1, lg.p, &tr, nullptr);
            for (int k = 0; k < nd; ++k) {
                const uint8_t* mk = blob<uint8_t>(tr, "dir" + std::to_string(k) + ".masks",
                                                  3 * static_cast<size_t>(L) * E) + static_cast<size_t>(L) * E;
                int prev = 0;
                for (int t = 0; t < L; ++t) {
                    int cnt = 0;
                    for (int ch = 0; ch < E; ++ch) cnt += mk[static_cast<size_t>(t) * E + ch];
                    const int after_refresh = refresh_at(t, cal.spec.n_refresh) ? 0 : prev;
                    out.timeline.push_back({"block" + std::to_string(blk) + ".dir" + std::to_string(k) + ".b_bar", t,
                                            after_refresh, cnt});
                    prev = cnt;
                }
            }
        }
    }
    m.spikes = SpikeCfg{};
    return out;
}

}  // namespace
}  // namespace ob

using ob::guarded;

extern "C" {

ouro_status ouro_b200_tensor_save(const char* path, int dtype, const uint64_t* shape, size_t rank, const void* data,
                                  int data_packed) {
    return guarded([&] {
        ob::require(path && (shape || rank == 0) && data, "tensor_save: NULL argument");
        ob::require(dtype >= 0 && dtype <= 2, "tensor_save: dtype must be 0 (f64), 1 (i8) or 2 (u4)");
        const std::vector<uint64_t> sh(shape, shape + rank);
        const auto dt = static_cast<ob::OuroDtype>(dtype);
        if (dt == ob::OuroDtype::U4 && !data_packed) {
            const size_t n = ob::ouro_numel(sh);
            std::vector<uint8_t> packed((n + 1) / 2);
            ob::pack_nibbles(static_cast<const int8_t*>(data), n, packed.data());
            ob::ouro_tensor_write(path, dt, sh, packed.data(), packed.size());
        } else {
            ob::ouro_tensor_write(path, dt, sh, data, ob::ouro_payload_bytes(dt, sh));
        }
    });
}

ouro_status ouro_b200_tensor_info(const char* path, int* dtype, uint64_t* shape, size_t cap, size_t* rank) {
    return guarded([&] {
        ob::require(path && dtype && rank, "tensor_info: NULL argument");
        const ob::OuroTensor t = ob::ouro_tensor_read(path);
        *dtype = static_cast<int>(t.dtype);
        *rank = t.shape.size();
        if (shape) std::copy(t.shape.begin(), t.shape.begin() + static_cast<long>(std::min(cap, t.shape.size())), shape);
    });
}

ouro_status ouro_b200_tensor_load(const char* path, int dtype, void* out, size_t cap, int out_packed) {
    return guarded([&] {
        ob::require(path && out, "tensor_load: NULL argument");
        const ob::OuroTensor t = ob::ouro_tensor_read(path);
        if (static_cast<int>(t.dtype) != dtype)
            throw ob::IoError(std::string(path) + ": dtype mismatch, file holds tag " +
                              std::to_string(static_cast<unsigned>(t.dtype)));
        if (t.dtype == ob::OuroDtype::U4 && !out_packed) {
            const size_t n = ob::ouro_numel(t.shape);
            ob::require(cap >= n, "tensor_load: output buffer too small");
            ob::unpack_nibbles(reinterpret_cast<const uint8_t*>(t.payload.data()), n, static_cast<int8_t*>(out));
        } else {
            ob::require(cap >= t.payload.size(), "tensor_load: output buffer too small");
            std::memcpy(out, t.payload.data(), t.payload.size());
        }
    });
}

ouro_status ouro_b200_quant_eval(const ouro_b200_stage_config* cfg, const char* calib_dir, const char* images_file,
                                 const char* out_dir) {
    return guarded([&] {
        ob::require(cfg != nullptr, "quant_eval: cfg is NULL");  // capi.cpp:177-182
        ob::require(calib_dir != nullptr, "quant_eval: calib_dir is NULL");
        ob::require(images_file != nullptr, "quant_eval: images_file is NULL");
        ob::require(out_dir != nullptr, "quant_eval: out_dir is NULL");
        const int mode = ob::mode_of(cfg->mode);
        const ob::QuantSpec spec = ob::spec_of(*cfg);
        ob::Context ctx(cfg->device);
        ob::Model m(&ctx, ob::make_toy_model(ob::dims_of(*cfg), {0, 1}, cfg->seed));
        ob::Calibration cal;
        cal.tokens = m.d.tokens();
        cal.embed = m.d.embed;
        cal.blocks = m.d.blocks;
        cal.ndirs = 2;
        cal.d1 = cfg->d1 != 0;
        ob::load_calibration_dir(cal, m.d.state, calib_dir, cfg->d2 != 0);
        ob::require(cal.spec.wbits == spec.wbits && cal.spec.abits == spec.abits && cal.spec.obits == spec.obits &&
                        cal.spec.n_refresh == spec.n_refresh && cal.spec.rho == spec.rho,
                    "calibration at " + std::string(calib_dir) +
                        " was made with different quantization settings than the config");  // pipeline.cpp:122-126
        const size_t pix = static_cast<size_t>(m.d.image) * m.d.image * m.d.channels;
        size_t file_batch = 0;
        std::vector<double> images = ob::load_images(images_file, pix, &file_batch);
        const size_t batch = std::min(file_batch, cfg->eval_batch);
        ob::require(batch >= 1, "quant_eval: eval_batch must be >= 1");
        images.resize(batch * pix);
        ob::SpikeCfg sp;
        if (cfg->spike_rate > 0.0) {
            ob::require(cfg->spike_channels >= 1 && cfg->spike_channels <= static_cast<size_t>(ob::kMaxSpikeChannels),
                        "quant_eval: spike_channels must be in [1, 64]");
            sp.rate = cfg->spike_rate;
            sp.gain = cfg->spike_gain;
            sp.channels = static_cast<int>(cfg->spike_channels);
            sp.salt = cfg->seed;  // spikes.salt = c.model.seed, pipeline.cpp:137
        }
        const ob::EvalOut r = ob::quant_eval(m, cal, mode, cfg->d1 != 0, cfg->d2 != 0, images,
                                             static_cast<int>(batch), sp);
        const std::string run = cfg->run_id ? cfg->run_id : "b200";
        ob::KV kv = {{"mode", cfg->mode},
                     {"weight_bits", std::to_string(cfg->weight_bits)},
                     {"act_bits", std::to_string(cfg->act_bits)},
                     {"outlier_bits", std::to_string(cfg->outlier_bits)},
                     {"batch", std::to_string(batch)},
                     {"logits_mse", ob::g17(r.logits_mse)},
                     {"argmax_agreement", ob::g17(static_cast<double>(r.argmax_agree) / static_cast<double>(batch))}};
        for (const auto& [name, mse] : r.layer_mse) kv.emplace_back("mse_" + name, mse);
        std::string metrics = ob::metrics_line(run, "quant-eval", kv);
        for (const auto& te : r.timeline)
            metrics += ob::metrics_line(run, "timeline", {{"tensor", te.tensor},
                                                          {"t", std::to_string(te.t)},
                                                          {"after_refresh", std::to_string(te.after_refresh)},
                                                          {"after_detect", std::to_string(te.after_detect)}});
        ob::ensure_dir(out_dir);
        const std::string od(out_dir);
        ob::atomic_write_bytes(od + "/metrics.txt", metrics);
        ob::atomic_write_bytes(od + "/manifest.txt", ob::manifest(*cfg, run, "quant-eval",
                                                                  {{"calibration", calib_dir},
                                                                   {"images_file", images_file}}));
    });
}

ouro_status ouro_b200_calib_stage(const ouro_b200_stage_config* cfg, const char* images_file, const char* out_dir) {
    return guarded([&] {
        ob::require(cfg != nullptr, "calib: cfg is NULL");  // capi.cpp:166-172
        ob::require(images_file != nullptr, "calib: images_file is NULL");
        ob::require(out_dir != nullptr, "calib: out_dir is NULL");
        const ob::QuantSpec spec = ob::spec_of(*cfg);
        ob::Context ctx(cfg->device);
        ob::Model m(&ctx, ob::make_toy_model(ob::dims_of(*cfg), {0, 1}, cfg->seed));
        const size_t pix = static_cast<size_t>(m.d.image) * m.d.image * m.d.channels;
        size_t batch = 0;
        const std::vector<double> images = ob::load_images(images_file, pix, &batch);
        ob::DevBuf<double> img;
        img.upload(images.data(), images.size(), ctx.stream);
        std::unique_ptr<ob::Calibration> cal =
            m.calibrate(img.p, static_cast<int>(batch), spec, cfg->d1 != 0, cfg->d2 != 0, 0);
        ob::ensure_dir(out_dir);
        ob::save_calibration_dir(*cal, m.d.state, out_dir);
        const std::string run = cfg->run_id ? cfg->run_id : "b200";
        ob::atomic_write_bytes(std::string(out_dir) + "/manifest.txt",
                               ob::manifest(*cfg, run, "calib",
                                            {{"images_file", images_file}, {"batch", std::to_string(batch)}}));
    });
}

}  // extern "C"
