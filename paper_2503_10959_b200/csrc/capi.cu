// C ABI (include/ouro_b200.h) over the engine and the K1-K4 launchers.
// Exception -> status mapping mirrors the reference's guarded()
// (/root/reference/proj/src/capi.cpp:18-37).
#include <cstring>
#include <exception>
#include <string>
#include <tuple>

#include "../../include/ouro_b200.h"
#include "engine.h"
#include "guard.h"
#include "planes.h"

using ob::require;

namespace ob {
std::string& last_error_slot() {
    static thread_local std::string slot;
    return slot;
}
}  // namespace ob
using ob::guarded;
#define g_last_error (ob::last_error_slot())

struct ouro_b200_ctx {
    std::unique_ptr<ob::Context> c;
};
struct ouro_b200_model {
    ouro_b200_ctx* ctx = nullptr;
    std::unique_ptr<ob::Model> m;
    bool graphs = false;
    // A captured graph bakes in raw pointers (workspace, weights, calibration
    // tables) and by-value kernel parameters (thresholds, literal routing), so
    // it is keyed on everything those depend on: the calibration's version (new
    // on create and on every edit; a freed-and-reallocated handle never matches),
    // the device allocation epoch (any DevBuf (re)allocation), and the call's
    // own arguments.
    struct GraphKey {
        const void* cal;
        uint64_t cal_version;
        int mode, d1, d2;
        const double* img;
        size_t B;
        double* logits;
        uint64_t epoch;
        bool operator==(const GraphKey& o) const {
            return std::tie(cal, cal_version, mode, d1, d2, img, B, logits, epoch) ==
                   std::tie(o.cal, o.cal_version, o.mode, o.d1, o.d2, o.img, o.B, o.logits, o.epoch);
        }
    };
    void drop_graphs() {
        if (exec) cudaGraphExecDestroy(exec);
        if (hexec) cudaGraphExecDestroy(hexec);
        exec = hexec = nullptr;
        key_hits = hkey_hits = 0;
    }
    GraphKey key{};
    int key_hits = 0;
    cudaGraphExec_t exec = nullptr;
    // end-to-end (host buffer) path: its own graph slot and the H2D copy stream
    GraphKey hkey{};
    int hkey_hits = 0;
    cudaGraphExec_t hexec = nullptr;
    cudaStream_t copy = nullptr;
    ~ouro_b200_model() {
        if (exec) cudaGraphExecDestroy(exec);
        if (hexec) cudaGraphExecDestroy(hexec);
        if (copy) cudaStreamDestroy(copy);
    }
};
struct ouro_b200_calib {
    std::unique_ptr<ob::Calibration> c;
};
struct ouro_b200_trace {
    ob::Model::TraceSink sink;
};

namespace {
// Capture `body` on stream st into a fresh executable graph (replacing *exec)
// and launch it once.
template <class Fn>
void capture_and_launch(cudaStream_t st, cudaGraphExec_t* exec, Fn&& body) {
    cudaGraph_t g = nullptr;
    ob::cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        body();
    } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    ob::cuda_check(cudaStreamEndCapture(st, &g), "end capture");
    if (*exec) cudaGraphExecDestroy(*exec);
    *exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(exec, g, 0);
    cudaGraphDestroy(g);
    ob::cuda_check(e, "graph instantiate");
    ob::cuda_check(cudaGraphLaunch(*exec, st), "graph launch");
}

// Graph policy shared by the device-buffer and host-buffer entry points: the
// first call with a key runs eagerly (it may allocate workspace or upload a
// calibration), the second identical call captures, later ones replay. The key's
// epoch is re-read after an eager run so allocations made by that run count.
template <class Fn>
void run_with_graph(ouro_b200_model* m, cudaStream_t st, ouro_b200_model::GraphKey key,
                    ouro_b200_model::GraphKey* slot, int* hits, cudaGraphExec_t* exec, Fn&& body) {
    if (!m->graphs || st == nullptr) {  // graphs need a capturable (non-legacy) stream
        body();
        return;
    }
    key.epoch = ob::alloc_epoch();
    if (*exec && *slot == key) {
        ob::cuda_check(cudaGraphLaunch(*exec, st), "graph launch");
        return;
    }
    if (*slot == key && *hits >= 1) {
        capture_and_launch(st, exec, body);
        require(ob::alloc_epoch() == key.epoch, "internal error: device memory was reallocated during graph capture");
        return;
    }
    if (*exec) {
        cudaGraphExecDestroy(*exec);
        *exec = nullptr;
    }
    body();
    key.epoch = ob::alloc_epoch();
    if (*slot == key) {
        ++*hits;
    } else {
        *slot = key;
        *hits = 1;
    }
}

bool is_pinned(const void* p) {
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, p) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();  // clear a benign "not a device pointer" status
    return pinned;
}
}  // namespace

extern "C" {

const char* ouro_b200_version(void) { return "0.1.0-sm100a"; }
const char* ouro_b200_last_error(void) { return g_last_error.c_str(); }

ouro_status ouro_b200_ctx_create(int device, ouro_b200_ctx** out) {
    return guarded([&] {
        require(out != nullptr, "ctx_create: out is NULL");
        auto h = std::make_unique<ouro_b200_ctx>();
        h->c = std::make_unique<ob::Context>(device);
        *out = h.release();
    });
}
void ouro_b200_ctx_free(ouro_b200_ctx* ctx) { delete ctx; }

ouro_status ouro_b200_ctx_set_stream(ouro_b200_ctx* ctx, void* stream) {
    return guarded([&] {
        require(ctx != nullptr, "ctx_set_stream: ctx is NULL");
        ctx->c->set_stream(static_cast<cudaStream_t>(stream));
    });
}
ouro_status ouro_b200_ctx_synchronize(ouro_b200_ctx* ctx) {
    return guarded([&] {
        require(ctx != nullptr, "ctx_synchronize: ctx is NULL");
        ob::cuda_check(cudaStreamSynchronize(ctx->c->stream), "synchronize");
    });
}
ouro_status ouro_b200_ctx_num_sms(ouro_b200_ctx* ctx, int* out) {
    return guarded([&] {
        require(ctx != nullptr && out != nullptr, "ctx_num_sms: NULL argument");
        *out = ctx->c->num_sms;
    });
}

static ouro_status detect_quantize_impl(ouro_b200_ctx* ctx, const double* x, const double* x2, const double* gate,
                                        size_t S, size_t T, size_t E, int src, int order, int grid, double theta,
                                        const double* s_in, const double* s_full, size_t n_refresh, unsigned act_bits,
                                        unsigned outlier_bits, int mode, int literal, int8_t* codes, uint8_t* codes4,
                                        double* s_row, int32_t* ocnt, uint32_t* omask, int8_t* ocode, double* oscale,
                                        uint8_t* scanned) {
    return guarded([&] {
        require(ctx && x && (codes || codes4) && s_row && ocnt && omask && ocode && oscale,
                "detect_quantize: NULL argument");
        require(!codes4 || (act_bits == 4 && E % 2 == 0),
                "detect_quantize_packed: packed codes need act_bits = 4 and an even channel count");
        require(mode == ob::MODE_DYNAMIC || mode == ob::MODE_STATIC, "detect_quantize: mode must be dynamic or static");
        require(mode == ob::MODE_STATIC ? s_full != nullptr : s_in != nullptr, "detect_quantize: missing scales");
        require(act_bits >= 2 && act_bits <= 8 && outlier_bits >= act_bits && outlier_bits <= 8,
                "detect_quantize: bit widths must satisfy 2 <= act <= outlier <= 8");
        require(src != ob::K1_SRC_MERGE || gate != nullptr, "detect_quantize: merge source needs the gate");
        require(src >= 0 && src <= 2, "detect_quantize: unknown source");
        require(literal >= 0 && literal <= 2, "detect_quantize: literal must be 0, 1 or 2");
        require(order >= -1 && order <= 3, "detect_quantize: order must be -1 (identity) or a scan order 0-3");
        require(order < 2 || (grid >= 1 && static_cast<size_t>(grid) * grid == T),
                "detect_quantize: column scan orders need T = grid^2");
        ob::K1Params k;
        k.S = static_cast<int>(S);
        k.T = static_cast<int>(T);
        k.E = static_cast<int>(E);
        k.src = src;
        k.x = x;
        k.x2 = x2;
        k.gate = gate;
        k.order = order;
        k.grid = grid;
        k.mode = mode;
        k.n_refresh = static_cast<int>(n_refresh);
        k.abits = act_bits;
        k.obits = outlier_bits;
        k.window = mode == ob::MODE_DYNAMIC ? (n_refresh > 0 ? static_cast<int>(n_refresh) : static_cast<int>(T)) : 8;
        k.cal.theta = theta;
        k.cal.s_in = s_in;
        k.cal.s_full = s_full;
        k.force_literal = literal == 1;
        k.window_kernel = literal == 2;
        k.codes = codes;
        k.codes4 = codes4;
        k.s_row = s_row;
        k.ocnt = ocnt;
        k.omask = omask;
        k.ocode = ocode;
        k.oscale = oscale;
        k.scanned = scanned;
        ob::cuda_check(ob::launch_k1(k, ctx->c->stream), "detect_quantize");
    });
}

ouro_status ouro_b200_detect_quantize(ouro_b200_ctx* ctx, const double* x, const double* x2, const double* gate,
                                      size_t S, size_t T, size_t E, int src, int order, int grid, double theta,
                                      const double* s_in, const double* s_full, size_t n_refresh, unsigned act_bits,
                                      unsigned outlier_bits, int mode, int literal, int8_t* codes, double* s_row,
                                      int32_t* ocnt, uint32_t* omask, int8_t* ocode, double* oscale,
                                      uint8_t* scanned, double* rs_work) {
    (void)rs_work;  // kept for ABI stability (round-1 signature); the row factor is computed in-kernel
    if (!codes) return guarded([] { throw ob::ValidationError("detect_quantize: NULL argument"); });
    return detect_quantize_impl(ctx, x, x2, gate, S, T, E, src, order, grid, theta, s_in, s_full, n_refresh, act_bits,
                                outlier_bits, mode, literal, codes, nullptr, s_row, ocnt, omask, ocode, oscale, scanned);
}

ouro_status ouro_b200_detect_quantize_packed(ouro_b200_ctx* ctx, const double* x, const double* x2, const double* gate,
                                             size_t S, size_t T, size_t E, int src, int order, int grid, double theta,
                                             const double* s_in, const double* s_full, size_t n_refresh,
                                             unsigned outlier_bits, int mode, int literal, uint8_t* codes4,
                                             double* s_row, int32_t* ocnt, uint32_t* omask, int8_t* ocode,
                                             double* oscale, uint8_t* scanned) {
    if (!codes4) return guarded([] { throw ob::ValidationError("detect_quantize_packed: NULL argument"); });
    return detect_quantize_impl(ctx, x, x2, gate, S, T, E, src, order, grid, theta, s_in, s_full, n_refresh, 4u,
                                outlier_bits, mode, literal, nullptr, codes4, s_row, ocnt, omask, ocode, oscale, scanned);
}

static ouro_status quant_linear_impl(ouro_b200_ctx* ctx, size_t M, size_t R, size_t K, const int8_t* codes,
                                     const uint8_t* codes4, const double* s_row, const int32_t* ocnt,
                                     const uint32_t* omask, const int8_t* ocode, const double* oscale, const int8_t* w,
                                     const int8_t* wt, const double* ws, int post, double* out, size_t ld_out,
                                     double* out2, size_t split, const double* bias, int32_t* acc_in,
                                     int32_t* acc_out) {
    return guarded([&] {
        require(ctx && (codes || codes4) && s_row && ocnt && omask && ocode && oscale && w && wt && ws && out,
                "quant_linear: NULL argument");
        require(K % 16 == 0 && R % 32 == 0, "quant_linear: K must be a multiple of 16 and R of 32");
        require(!codes4 || K % 32 == 0, "quant_linear_packed: K must be a multiple of 32");
        require((acc_in == nullptr) == (acc_out == nullptr), "quant_linear: acc_in and acc_out go together");
        require(post != ob::POST_INPROJ || (out2 != nullptr && split % 32 == 0 && split < R),
                "quant_linear: in_proj post-op needs out2 and a split that is a multiple of 32");
        require(post != ob::POST_BIAS, "quant_linear: bias post-op is not part of the hybrid epilogue");
        require(post != ob::POST_XPROJ || (bias != nullptr && split <= R), "quant_linear: x_proj post-op needs bias");
        ob::QLinParams q;
        q.M = static_cast<int>(M);
        q.R = static_cast<int>(R);
        q.K = static_cast<int>(K);
        q.a.codes = const_cast<int8_t*>(codes);
        q.a.codes4 = const_cast<uint8_t*>(codes4);
        q.a.s_row = const_cast<double*>(s_row);
        q.a.ocnt = const_cast<int*>(ocnt);
        q.a.omask = const_cast<uint32_t*>(omask);
        q.a.ocode = const_cast<int8_t*>(ocode);
        q.a.oscale = const_cast<double*>(oscale);
        q.a.J = static_cast<int>((K + 31) / 32);
        q.w = w;
        q.wt = wt;
        q.ws = ws;
        q.epi.post = post;
        q.epi.out = out;
        q.epi.ld_out = static_cast<int>(ld_out);
        q.epi.out2 = out2;
        q.epi.split = static_cast<int>(split);
        q.epi.bias = bias;
        q.epi.acc_in = acc_in;
        q.epi.acc_out = acc_out;
        ob::cuda_check(ob::launch_qlinear(q, ctx->c->stream, ctx->c->num_sms), "quant_linear");
    });
}

ouro_status ouro_b200_quant_linear(ouro_b200_ctx* ctx, size_t M, size_t R, size_t K, const int8_t* codes,
                                   const double* s_row, const int32_t* ocnt, const uint32_t* omask,
                                   const int8_t* ocode, const double* oscale, const int8_t* w, const int8_t* wt,
                                   const double* ws, int post, double* out, size_t ld_out, double* out2, size_t split,
                                   const double* bias, int32_t* acc_in, int32_t* acc_out) {
    if (!codes) return guarded([] { throw ob::ValidationError("quant_linear: NULL argument"); });
    return quant_linear_impl(ctx, M, R, K, codes, nullptr, s_row, ocnt, omask, ocode, oscale, w, wt, ws, post, out,
                             ld_out, out2, split, bias, acc_in, acc_out);
}

ouro_status ouro_b200_quant_linear_packed(ouro_b200_ctx* ctx, size_t M, size_t R, size_t K, const uint8_t* codes4,
                                          const double* s_row, const int32_t* ocnt, const uint32_t* omask,
                                          const int8_t* ocode, const double* oscale, const int8_t* w,
                                          const int8_t* wt, const double* ws, int post, double* out, size_t ld_out,
                                          double* out2, size_t split, const double* bias, int32_t* acc_in,
                                          int32_t* acc_out) {
    if (!codes4) return guarded([] { throw ob::ValidationError("quant_linear_packed: NULL argument"); });
    return quant_linear_impl(ctx, M, R, K, nullptr, codes4, s_row, ocnt, omask, ocode, oscale, w, wt, ws, post, out,
                             ld_out, out2, split, bias, acc_in, acc_out);
}

static void quant_scan_impl(ouro_b200_ctx* ctx, size_t S, size_t T, size_t E, size_t N, int order, int grid,
                            const double* u, const double* proj, const double* a, const double* b_delta, double* o,
                            int mode, size_t n_refresh, unsigned act_bits, unsigned outlier_bits, const double* theta,
                            const double* const* s_in, const double* const* s_full, const uint8_t* literal,
                            int force_literal, uint8_t* masks, const ob::SpikeCfg& spike) {
    require(ctx && u && proj && a && b_delta && o, "quant_scan: NULL argument");
    require(N == 16, "quant_scan: this build keeps N = 16 states per channel");
    require(mode == ob::MODE_FP || (theta && s_in && s_full), "quant_scan: quantized modes need calibration");
    require(order >= 0 && order <= 3, "quant_scan: order must be a scan order 0-3");
    require(order < 2 || (grid >= 1 && static_cast<size_t>(grid) * grid == T),
            "quant_scan: column scan orders need T = grid^2");
    ob::ScanParams p;
    p.S = static_cast<int>(S);
    p.T = static_cast<int>(T);
    p.E = static_cast<int>(E);
    p.N = static_cast<int>(N);
    p.order = order;
    p.grid = grid;
    p.u = u;
    p.proj = proj;
    p.a = a;
    p.b_delta = b_delta;
    p.o = o;
    p.mode = mode;
    p.n_refresh = static_cast<int>(n_refresh);
    p.abits = act_bits;
    p.obits = outlier_bits;
    if (mode != ob::MODE_FP)
        for (int k = 0; k < 3; ++k) {
            p.cal[k].theta = theta[k];
            p.cal[k].s_in = s_in[k];
            p.cal[k].s_full = s_full[k];
        }
    p.literal = literal;
    p.literal_any = literal != nullptr ? 1 : 0;
    p.force_literal = force_literal;
    p.masks = masks;
    p.spike = spike;
    ob::cuda_check(ob::launch_scan(p, ctx->c->stream, nullptr), "quant_scan");
}

static ob::SpikeCfg spike_from(const ouro_b200_spikes* sp) {
    ob::SpikeCfg c;
    if (sp == nullptr || !(sp->rate > 0.0)) return c;
    require(sp->channels >= 1 && sp->channels <= static_cast<size_t>(ob::kMaxSpikeChannels),
            "spikes: channels must be in [1, 64]");
    c.rate = sp->rate;
    c.gain = sp->gain;
    c.channels = static_cast<int>(sp->channels);
    c.salt = sp->salt;
    c.sample0 = static_cast<int>(sp->sample0);
    return c;
}

ouro_status ouro_b200_quant_scan(ouro_b200_ctx* ctx, size_t S, size_t T, size_t E, size_t N, int order, int grid,
                                 const double* u, const double* proj, const double* a, const double* b_delta,
                                 double* o, int mode, size_t n_refresh, unsigned act_bits, unsigned outlier_bits,
                                 const double* theta, const double* const* s_in, const double* const* s_full,
                                 const uint8_t* literal, int force_literal, uint8_t* masks) {
    return guarded([&] {
        quant_scan_impl(ctx, S, T, E, N, order, grid, u, proj, a, b_delta, o, mode, n_refresh, act_bits,
                        outlier_bits, theta, s_in, s_full, literal, force_literal, masks, ob::SpikeCfg{});
    });
}

ouro_status ouro_b200_quant_scan_spiked(ouro_b200_ctx* ctx, size_t S, size_t T, size_t E, size_t N, int order,
                                        int grid, const double* u, const double* proj, const double* a,
                                        const double* b_delta, double* o, int mode, size_t n_refresh,
                                        unsigned act_bits, unsigned outlier_bits, const double* theta,
                                        const double* const* s_in, const double* const* s_full,
                                        const ouro_b200_spikes* spikes, size_t block, size_t dir, size_t sample0) {
    return guarded([&] {
        ob::SpikeCfg c = spike_from(spikes);
        c.block = static_cast<int>(block);
        c.dir = static_cast<int>(dir);
        c.sample0 += static_cast<int>(sample0);
        quant_scan_impl(ctx, S, T, E, N, order, grid, u, proj, a, b_delta, o, mode, n_refresh, act_bits,
                        outlier_bits, theta, s_in, s_full, nullptr, 0, nullptr, c);
    });
}

ouro_status ouro_b200_dgemm(ouro_b200_ctx* ctx, size_t M, size_t R, size_t K, const double* a, size_t lda,
                            const double* w, int post, double* out, size_t ld_out, double* out2, size_t split,
                            const double* bias) {
    return guarded([&] {
        require(ctx && a && w && out, "dgemm: NULL argument");
        ob::DGemmParams g;
        g.M = static_cast<int>(M);
        g.R = static_cast<int>(R);
        g.K = static_cast<int>(K);
        g.a = a;
        g.lda = static_cast<int>(lda);
        g.w = w;
        g.epi.post = post;
        g.epi.out = out;
        g.epi.ld_out = static_cast<int>(ld_out);
        g.epi.out2 = out2;
        g.epi.split = static_cast<int>(split);
        g.epi.bias = bias;
        ob::cuda_check(ob::launch_dgemm(g, ctx->c->stream), "dgemm");
    });
}

ouro_status ouro_b200_model_create(ouro_b200_ctx* ctx, const size_t* dims, const int* orders, size_t ndirs,
                                   uint64_t seed, ouro_b200_model** out) {
    return guarded([&] {
        require(ctx && dims && orders && out, "model_create: NULL argument");
        ob::Dims d;
        d.image = static_cast<int>(dims[0]);
        d.channels = static_cast<int>(dims[1]);
        d.patch = static_cast<int>(dims[2]);
        d.embed = static_cast<int>(dims[3]);
        d.state = static_cast<int>(dims[4]);
        d.blocks = static_cast<int>(dims[5]);
        d.classes = static_cast<int>(dims[6]);
        d.conv_width = static_cast<int>(dims[7]);
        auto h = std::make_unique<ouro_b200_model>();
        h->ctx = ctx;
        h->m = std::make_unique<ob::Model>(ctx->c.get(),
                                           ob::make_toy_model(d, std::vector<int>(orders, orders + ndirs), seed));
        *out = h.release();
    });
}
void ouro_b200_model_free(ouro_b200_model* m) { delete m; }

ouro_status ouro_b200_model_set_tensor(ouro_b200_model* m, const char* name, const double* host, size_t n) {
    return guarded([&] {
        require(m && name && host, "model_set_tensor: NULL argument");
        m->m->set_tensor(name, host, n);
        m->drop_graphs();  // weights are uploaded by forward()'s host code, which a replay skips
    });
}
ouro_status ouro_b200_model_get_tensor(ouro_b200_model* m, const char* name, double* host, size_t cap,
                                       size_t* n_out) {
    return guarded([&] {
        require(m && name, "model_get_tensor: NULL argument");
        auto it = m->m->host.t.find(name);
        require(it != m->m->host.t.end(), std::string("model_get_tensor: unknown tensor '") + name + "'");
        if (n_out) *n_out = it->second.size();
        if (host) std::memcpy(host, it->second.data(), std::min(cap, it->second.size()) * sizeof(double));
    });
}

static ob::QuantSpec spec_from(const unsigned* bits, size_t n_refresh, double rho) {
    ob::QuantSpec s;
    s.wbits = bits[0];
    s.abits = bits[1];
    s.obits = bits[2];
    s.n_refresh = static_cast<int>(n_refresh);
    s.rho = rho;
    s.validate();
    require(s.abits <= 8, "activation bits above 8 do not fit the int8 operand");
    require(s.wbits <= 4, "weight codes must fit the int4 range (bits <= 4)");
    return s;
}

ouro_status ouro_b200_model_get_qweight(ouro_b200_model* m, const char* name, unsigned bits, double* out,
                                       size_t cap, size_t* n) {
    return guarded([&] {
        require(m && name && n, "model_get_qweight: NULL argument");
        require(bits >= 2 && bits <= 8, "model_get_qweight: bits must be in [2, 8]");
        const std::vector<double> v = m->m->host.dequantized(name, bits);
        *n = v.size();
        if (out) {
            require(cap >= v.size(), "model_get_qweight: output buffer too small");
            std::memcpy(out, v.data(), v.size() * sizeof(double));
        }
    });
}

ouro_status ouro_b200_calib_create(ouro_b200_model* m, const unsigned* bits, size_t n_refresh, double rho, int d1,
                                   int d2, ouro_b200_calib** out) {
    return guarded([&] {
        require(m && bits && out, "calib_create: NULL argument");
        auto h = std::make_unique<ouro_b200_calib>();
        h->c = std::make_unique<ob::Calibration>();
        ob::Calibration& c = *h->c;
        const ob::Dims& d = m->m->d;
        c.spec = spec_from(bits, n_refresh, rho);
        c.d1 = d1 != 0;
        c.d2 = d2 != 0;
        c.tokens = d.tokens();
        c.embed = d.embed;
        c.blocks = d.blocks;
        c.ndirs = static_cast<int>(m->m->host.orders.size());
        ob::TensorCal z;
        z.s_in.assign(c.tokens, 1.0);
        z.s_full.assign(c.tokens, 1.0);
        z.excluded.assign(c.embed, 0);
        c.scan.assign(static_cast<size_t>(c.blocks) * c.ndirs * 3, z);
        if (c.d2) c.lin.assign(static_cast<size_t>(c.blocks) * c.nsites(), z);
        *out = h.release();
    });
}

ouro_status ouro_b200_calibrate(ouro_b200_model* m, const double* images_dev, size_t B, const unsigned* bits,
                                size_t n_refresh, double rho, int d1, int d2, size_t chunk, ouro_b200_calib** out) {
    return guarded([&] {
        require(m && images_dev && bits && out, "calibrate: NULL argument");
        require(B >= 1, "calibrate: need at least one image");
        auto h = std::make_unique<ouro_b200_calib>();
        h->c = m->m->calibrate(images_dev, static_cast<int>(B), spec_from(bits, n_refresh, rho), d1 != 0, d2 != 0,
                               static_cast<int>(chunk));
        *out = h.release();
    });
}
void ouro_b200_calib_free(ouro_b200_calib* c) { delete c; }

ouro_status ouro_b200_calib_save(ouro_b200_calib* c, ouro_b200_model* m, const char* dir) {
    return guarded([&] {
        require(c && m && dir, "calib_save: NULL argument");
        ob::save_calibration_dir(*c->c, m->m->d.state, dir);
    });
}

ouro_status ouro_b200_calib_load(ouro_b200_model* m, const char* dir, int d1, int d2, ouro_b200_calib** out) {
    return guarded([&] {
        require(m && dir && out, "calib_load: NULL argument");
        auto h = std::make_unique<ouro_b200_calib>();
        h->c = std::make_unique<ob::Calibration>();
        ob::Calibration& c = *h->c;
        const ob::Dims& d = m->m->d;
        c.d1 = d1 != 0;
        c.tokens = d.tokens();
        c.embed = d.embed;
        c.blocks = d.blocks;
        c.ndirs = static_cast<int>(m->m->host.orders.size());
        ob::load_calibration_dir(c, d.state, dir, d2 != 0);
        require(c.spec.abits <= 8 && c.spec.wbits <= 4, "calib_load: bit widths outside this build's operands");
        *out = h.release();
    });
}

ouro_status ouro_b200_calib_spec(ouro_b200_calib* c, unsigned* bits, size_t* n_refresh, double* rho, int* d1,
                                 int* d2) {
    return guarded([&] {
        require(c && bits && n_refresh && rho && d1 && d2, "calib_spec: NULL argument");
        const ob::Calibration& k = *c->c;
        bits[0] = k.spec.wbits;
        bits[1] = k.spec.abits;
        bits[2] = k.spec.obits;
        *n_refresh = static_cast<size_t>(k.spec.n_refresh);
        *rho = k.spec.rho;
        *d1 = k.d1 ? 1 : 0;
        *d2 = k.d2 ? 1 : 0;
    });
}

ouro_status ouro_b200_calib_count(ouro_b200_calib* c, int which, size_t* out) {
    return guarded([&] {
        require(c && out, "calib_count: NULL argument");
        *out = which == 0 ? c->c->scan.size() : c->c->lin.size();
    });
}
ouro_status ouro_b200_calib_get(ouro_b200_calib* c, int which, size_t idx, double* theta, double* s_in,
                                double* s_full, uint8_t* excluded) {
    return guarded([&] {
        require(c != nullptr, "calib_get: calib is NULL");
        auto& v = which == 0 ? c->c->scan : c->c->lin;
        require(idx < v.size(), "calib_get: index out of range");
        const ob::TensorCal& t = v[idx];
        if (theta) *theta = t.theta;
        if (s_in) std::memcpy(s_in, t.s_in.data(), t.s_in.size() * sizeof(double));
        if (s_full) std::memcpy(s_full, t.s_full.data(), t.s_full.size() * sizeof(double));
        if (excluded) std::memcpy(excluded, t.excluded.data(), t.excluded.size());
    });
}
ouro_status ouro_b200_calib_set(ouro_b200_calib* c, int which, size_t idx, double theta, const double* s_in,
                                const double* s_full, const uint8_t* excluded) {
    return guarded([&] {
        require(c != nullptr, "calib_set: calib is NULL");
        auto& v = which == 0 ? c->c->scan : c->c->lin;
        require(idx < v.size(), "calib_set: index out of range");
        ob::TensorCal& t = v[idx];
        t.theta = theta;
        if (s_in) std::memcpy(t.s_in.data(), s_in, t.s_in.size() * sizeof(double));
        if (s_full) std::memcpy(t.s_full.data(), s_full, t.s_full.size() * sizeof(double));
        if (excluded) std::memcpy(t.excluded.data(), excluded, t.excluded.size());
        c->c->dirty = true;
        c->c->version = ob::next_calib_version();
    });
}

ouro_status ouro_b200_model_use_graphs(ouro_b200_model* m, int on) {
    return guarded([&] {
        require(m != nullptr, "model_use_graphs: model is NULL");
        m->graphs = on != 0;
        if (!m->graphs) m->drop_graphs();
    });
}


ouro_status ouro_b200_forward(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                              const double* images_dev, size_t B, double* logits_dev) {
    return guarded([&] {
        require(m && images_dev && logits_dev, "forward: NULL argument");
        require(mode == ob::MODE_FP || c != nullptr, "forward: quantized modes need a calibration");
        ob::Calibration* cal = c ? c->c.get() : nullptr;
        cudaStream_t st = m->ctx->c->stream;
        ouro_b200_model::GraphKey key{cal, cal ? cal->version : 0, mode, d1, d2, images_dev, B, logits_dev, 0};
        run_with_graph(m, st, key, &m->key, &m->key_hits, &m->exec, [&] {
            m->m->forward(cal, mode, d1 != 0, d2 != 0, images_dev, static_cast<int>(B), logits_dev, nullptr,
                          nullptr);
        });
    });
}

ouro_status ouro_b200_forward_host(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                   const double* images_host, size_t B, double* logits_host) {
    return guarded([&] {
        require(m && images_host && logits_host, "forward_host: NULL argument");
        require(mode == ob::MODE_FP || c != nullptr, "forward_host: quantized modes need a calibration");
        ob::Model& mm = *m->m;
        ob::Calibration* cal = c ? c->c.get() : nullptr;
        const size_t pix = static_cast<size_t>(mm.d.image) * mm.d.image * mm.d.channels;
        cudaStream_t st = m->ctx->c->stream;
        mm.w.img.ensure(B * pix);
        mm.w.logits.ensure(B * mm.d.classes);
        const size_t lbytes = B * mm.d.classes * sizeof(double);
        // The overlapped (and capturable) path needs both host buffers pinned: a
        // pageable copy can neither overlap nor be captured into a graph.
        if (!is_pinned(images_host) || !is_pinned(logits_host) || st == nullptr) {
            ob::cuda_check(cudaMemcpyAsync(mm.w.img.p, images_host, B * pix * sizeof(double), cudaMemcpyHostToDevice, st),
                           "H2D images");
            ouro_status s = ouro_b200_forward(m, c, mode, d1, d2, mm.w.img.p, B, mm.w.logits.p);
            if (s != OURO_OK) throw ob::ValidationError(g_last_error);
            ob::cuda_check(cudaMemcpyAsync(logits_host, mm.w.logits.p, lbytes, cudaMemcpyDeviceToHost, st), "D2H logits");
            ob::cuda_check(cudaStreamSynchronize(st), "forward_host sync");
            return;
        }
        if (!m->copy) ob::cuda_check(cudaStreamCreateWithFlags(&m->copy, cudaStreamNonBlocking), "copy stream");
        // pinned images: the H2D copy runs in chunks on the copy stream, each chunk's
        // patch gather + embedding waits only for its own chunk (Model::HostFeed)
        ob::Model::HostFeed feed;
        feed.host = images_host;
        feed.copy = m->copy;
        feed.chunks = B >= 64 ? m->m->feed_chunks : 1;
        ouro_b200_model::GraphKey key{cal, cal ? cal->version : 0, mode, d1, d2, images_host, B, logits_host, 0};
        run_with_graph(m, st, key, &m->hkey, &m->hkey_hits, &m->hexec, [&] {
            mm.forward(cal, mode, d1 != 0, d2 != 0, mm.w.img.p, static_cast<int>(B), mm.w.logits.p, nullptr, nullptr,
                       &feed);
            ob::cuda_check(cudaMemcpyAsync(logits_host, mm.w.logits.p, lbytes, cudaMemcpyDeviceToHost, st), "D2H logits");
        });
        ob::cuda_check(cudaStreamSynchronize(st), "forward_host sync");
    });
}

ouro_status ouro_b200_model_set_spikes(ouro_b200_model* m, const ouro_b200_spikes* spikes) {
    return guarded([&] {
        require(m != nullptr, "model_set_spikes: model is NULL");
        m->m->spikes = spike_from(spikes);
        m->drop_graphs();
    });
}

ouro_status ouro_b200_model_set_option(ouro_b200_model* m, const char* key, long value) {
    return guarded([&] {
        require(m && key, "model_set_option: NULL argument");
        const std::string k(key);
        if (k == "scan_variant") {
            require(value >= 0 && value <= 7, "model_set_option: scan_variant must be 0..7");
            m->m->scan_variant = static_cast<int>(value);
        } else if (k == "feed_chunks") {
            require(value >= 1 && value <= 64, "model_set_option: feed_chunks must be in [1, 64]");
            m->m->feed_chunks = static_cast<int>(value);
        } else if (k == "split_min_rows") {
            require(value >= 0, "model_set_option: split_min_rows must be >= 0");
            m->m->split_min_rows = static_cast<int>(value);
        } else if (k == "split_parts") {
            require(value >= 1 && value <= 4, "model_set_option: split_parts must be in [1, 4]");
            m->m->split_parts = static_cast<int>(value);
        } else if (k == "merge_fuse") {
            require(value == 0 || value == 1, "model_set_option: merge_fuse must be 0 or 1");
            m->m->merge_fuse = static_cast<int>(value);
        } else if (k == "pack_a4") {
            require(value == 0 || value == 1, "model_set_option: pack_a4 must be 0 or 1");
            m->m->pack_a4 = static_cast<int>(value);
        } else if (k == "k1_variant") {
            require(value >= 0 && value <= 2, "model_set_option: k1_variant must be 0, 1 or 2");
            m->m->k1_variant = static_cast<int>(value);
        } else {
            throw ob::ValidationError("model_set_option: unknown option '" + k + "'");
        }
        m->drop_graphs();
    });
}

ouro_status ouro_b200_forward_profile(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                      const double* images_dev, size_t B, double* logits_dev, double* ms,
                                      int* launches) {
    return guarded([&] {
        require(m && images_dev && logits_dev && ms && launches, "forward_profile: NULL argument");
        require(mode == ob::MODE_FP || c != nullptr, "forward_profile: quantized modes need a calibration");
        ob::Model& mm = *m->m;
        mm.timing = ob::Model::Timing{};
        mm.timing.on = true;
        try {
            mm.forward(c ? c->c.get() : nullptr, mode, d1 != 0, d2 != 0, images_dev, static_cast<int>(B), logits_dev,
                       nullptr, nullptr);
        } catch (...) {
            mm.timing.on = false;
            throw;
        }
        mm.timing_collect();
        mm.timing.on = false;
        for (int i = 0; i < ob::Model::FAM_COUNT; ++i) {
            ms[i] = mm.timing.ms[i];
            launches[i] = mm.timing.launches[i];
        }
    });
}

ouro_status ouro_b200_forward_profile_launches(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                               const double* images_dev, size_t B, double* logits_dev, double* ms,
                                               int* family, size_t cap, size_t* n) {
    return guarded([&] {
        require(m && images_dev && logits_dev && ms && family && n, "forward_profile_launches: NULL argument");
        ob::Model& mm = *m->m;
        mm.timing = ob::Model::Timing{};
        mm.timing.on = true;
        mm.timing.keep_list = true;
        try {
            mm.forward(c ? c->c.get() : nullptr, mode, d1 != 0, d2 != 0, images_dev, static_cast<int>(B), logits_dev,
                       nullptr, nullptr);
        } catch (...) {
            mm.timing.on = false;
            throw;
        }
        mm.timing_collect();
        mm.timing.on = false;
        *n = mm.timing.list.size();
        for (size_t k = 0; k < std::min(cap, mm.timing.list.size()); ++k) {
            family[k] = mm.timing.list[k].first;
            ms[k] = mm.timing.list[k].second;
        }
    });
}

ouro_status ouro_b200_measure_fp64_peak(ouro_b200_ctx* ctx, double* tflops) {
    return guarded([&] {
        require(ctx && tflops, "measure_fp64_peak: NULL argument");
        *tflops = ob::measure_fp64_peak(ctx->c->stream, ctx->c->num_sms);
    });
}

ouro_status ouro_b200_launch_count(long long* out) {
    return guarded([&] {
        require(out != nullptr, "launch_count: out is NULL");
        *out = ob::kernel_launch_counter();
    });
}

ouro_status ouro_b200_measure_i8_peak(ouro_b200_ctx* ctx, double* tops) {
    return guarded([&] {
        require(ctx && tops, "measure_i8_peak: NULL argument");
        *tops = ob::measure_i8_peak(ctx->c->stream, ctx->c->num_sms);
        ob::require(*tops > 0.0, "measure_i8_peak: probe failed");
    });
}

ouro_status ouro_b200_detect_quantize_planes(ouro_b200_ctx* ctx, const double* x, size_t steps, size_t K, size_t C,
                                             double theta, const double* s_in, size_t n_refresh, unsigned act_bits,
                                             unsigned outlier_bits, size_t Kp, int8_t* codes, double* s_row,
                                             int32_t* ocnt, uint32_t* omask, int8_t* ocode, double* oscale,
                                             uint8_t* scanned) {
    return guarded([&] {
        require(ctx && x && s_in && codes && s_row && ocnt && omask && ocode && oscale,
                "detect_quantize_planes: NULL argument");
        require(steps >= 1 && C >= 1 && K >= 1 && K <= 4096, "detect_quantize_planes: need steps, C >= 1 and 1 <= K <= 4096");
        require(Kp >= K && Kp <= (1u << 20), "detect_quantize_planes: Kp must be >= K");
        require(steps * C <= static_cast<size_t>(INT32_MAX) && steps <= 65535, "detect_quantize_planes: too many rows");
        require(act_bits >= 2 && act_bits <= outlier_bits && outlier_bits <= 8,
                "detect_quantize_planes: need 2 <= act_bits <= outlier_bits <= 8");
        ob::PlaneParams p;
        p.x = x;
        p.steps = static_cast<int>(steps);
        p.K = static_cast<int>(K);
        p.Kp = static_cast<int>(Kp);
        p.C = static_cast<int>(C);
        p.theta = theta;
        p.s_in = s_in;
        p.n_refresh = static_cast<int>(n_refresh);
        p.abits = static_cast<int>(act_bits);
        p.obits = static_cast<int>(outlier_bits);
        p.a = ob::QAct{codes, nullptr, s_row, ocnt, omask, ocode, oscale, static_cast<int>((Kp + 31) / 32)};
        p.scanned = scanned;
        void* work = nullptr;
        cudaStream_t st = ctx->c->stream;
        ob::cuda_check(cudaMallocAsync(&work, ob::plane_workspace_bytes(p.steps, p.K), st), "workspace");
        p.work = work;
        const cudaError_t e = ob::launch_detect_planes(p, st);
        cudaFreeAsync(work, st);
        ob::cuda_check(e, "detect_quantize_planes");
    });
}

ouro_status ouro_b200_refresh_sweep(ouro_b200_ctx* ctx, const ouro_b200_sweep_settings* s,
                                    ouro_b200_sweep_record* records, double* outputs) {
    return guarded([&] {
        require(ctx && s && records && (s->periods || s->n_periods == 0), "refresh_sweep: NULL argument");
        ob::SweepSettings ss;
        ss.periods.assign(s->periods, s->periods + s->n_periods);
        ss.steps = s->steps;
        ss.m = s->m;
        ss.k = s->k;
        ss.c = s->c;
        ss.persistent_channels = s->persistent_channels;
        ss.transient_rate = s->transient_rate;
        ss.spike_gain = s->spike_gain;
        ss.trials = s->trials;
        ss.seed = s->seed;
        std::vector<double> y;
        const auto recs = ob::refresh_sweep(ss, ctx->c->stream, ctx->c->num_sms, outputs ? &y : nullptr);
        for (size_t i = 0; i < recs.size(); ++i)
            records[i] = {recs[i].period, recs[i].median_total_ns, recs[i].mean_o_list, recs[i].scans_per_step};
        if (outputs) std::memcpy(outputs, y.data(), y.size() * sizeof(double));
    });
}

ouro_status ouro_b200_gemm_bench(ouro_b200_ctx* ctx, const ouro_b200_bench_settings* s,
                                 ouro_b200_bench_record* records) {
    return guarded([&] {
        require(ctx && s && records && (s->sizes || s->n_sizes == 0), "gemm_bench: NULL argument");
        ob::BenchSettings bs;
        bs.sizes.assign(s->sizes, s->sizes + s->n_sizes);
        bs.outlier_fraction = s->outlier_fraction;
        bs.trials = s->trials;
        bs.seed = s->seed;
        bs.f16_output = s->f16_output != 0;
        const auto recs = ob::gemm_bench(bs, ctx->c->stream, ctx->c->num_sms);
        for (size_t i = 0; i < recs.size(); ++i)
            records[i] = {recs[i].path == "hybrid" ? 0 : 1, recs[i].size, recs[i].median_ns};
    });
}

ouro_status ouro_b200_math_eval(ouro_b200_ctx* ctx, int fn, const double* x_dev, double* y_dev, size_t n) {
    return guarded([&] {
        require(ctx != nullptr, "math_eval: ctx is NULL");
        require(fn >= 0 && fn <= 3, "math_eval: fn must be 0 (exp), 1 (log1p), 2 (softplus) or 3 (silu)");
        require(n == 0 || (x_dev && y_dev), "math_eval: NULL buffer");
        ob::cuda_check(ob::launch_math_eval(fn, x_dev, y_dev, n, ctx->c->stream), "math_eval");
    });
}

ouro_status ouro_b200_trace_run(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                const double* images_host, size_t B, size_t block, ouro_b200_trace** out) {
    return guarded([&] {
        require(m && images_host && out, "trace_run: NULL argument");
        require(mode == ob::MODE_FP || c != nullptr, "trace_run: quantized modes need a calibration");
        ob::Model& mm = *m->m;
        require(block < static_cast<size_t>(mm.d.blocks), "trace_run: block out of range");
        const size_t pix = static_cast<size_t>(mm.d.image) * mm.d.image * mm.d.channels;
        cudaStream_t st = m->ctx->c->stream;
        ob::DevBuf<double> img, logits;
        img.upload(images_host, B * pix, st);
        logits.ensure(B * mm.d.classes);
        auto h = std::make_unique<ouro_b200_trace>();
        h->sink.block = static_cast<int>(block);
        mm.forward(c ? c->c.get() : nullptr, mode, d1 != 0, d2 != 0, img.p, static_cast<int>(B), logits.p, &h->sink,
                   nullptr);
        std::vector<char> lb(B * mm.d.classes * sizeof(double));
        ob::cuda_check(cudaStreamSynchronize(st), "trace sync");
        ob::cuda_check(cudaMemcpy(lb.data(), logits.p, lb.size(), cudaMemcpyDeviceToHost), "trace logits");
        h->sink.blobs["logits"] = std::move(lb);
        *out = h.release();
    });
}
ouro_status ouro_b200_trace_get(ouro_b200_trace* t, const char* key, void* host, size_t cap, size_t* bytes) {
    return guarded([&] {
        require(t && key, "trace_get: NULL argument");
        auto it = t->sink.blobs.find(key);
        require(it != t->sink.blobs.end(), std::string("trace_get: no entry '") + key + "'");
        if (bytes) *bytes = it->second.size();
        if (host) std::memcpy(host, it->second.data(), std::min(cap, it->second.size()));
    });
}
void ouro_b200_trace_free(ouro_b200_trace* t) { delete t; }

}  // extern "C"
