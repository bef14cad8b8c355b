// Host engine: weights, calibration tables and the forward schedule.
// Every arithmetic step of the forward runs in the K1-K4 kernels; the host
// only prepares weights (W4 row quantization, once per model, quant.cpp:355-402),
// reduces calibration statistics (quantile, quant.cpp:117-177) and launches.
#include <atomic>
#include "engine.h"
#include "seeded_rng.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>

namespace ob {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        const bool launch_cfg = e == cudaErrorInvalidValue || e == cudaErrorInvalidConfiguration;
        std::string m = std::string(what) + ": " + cudaGetErrorString(e);
        if (launch_cfg) throw ValidationError(m);
        throw NumericError(m);
    }
}

void QuantSpec::validate() const {  // quant.cpp:54-60
    require(wbits >= 2, "weight bits must be >= 2");
    require(abits >= 2, "activation bits must be >= 2");
    require(obits >= 2 && obits <= 8, "outlier bits must be in [2, 8]");
    require(abits <= obits, "inlier activation bits must not exceed outlier bits");
    require(rho >= 0.0 && rho < 1.0, "rho must be in [0, 1)");
    require(n_refresh >= 0, "n_refresh must be >= 0");
}

namespace {
std::atomic<uint64_t> g_alloc_epoch{1};
std::atomic<uint64_t> g_calib_version{1};
}  // namespace
uint64_t alloc_epoch() { return g_alloc_epoch.load(std::memory_order_acquire); }
uint64_t next_calib_version() { return g_calib_version.fetch_add(1, std::memory_order_relaxed); }

template <class T>
void DevBuf<T>::release() {
    if (p) {
        cudaFree(p);
        g_alloc_epoch.fetch_add(1, std::memory_order_release);
    }
    p = nullptr;
    n = 0;
}
template <class T>
void DevBuf<T>::ensure(size_t count) {
    if (count <= n) return;
    release();
    cuda_check(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    g_alloc_epoch.fetch_add(1, std::memory_order_release);
    n = count;
}
template <class T>
void DevBuf<T>::upload(const T* host, size_t count, cudaStream_t st) {
    ensure(count);
    cuda_check(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
}
template struct DevBuf<double>;
template struct DevBuf<int8_t>;
template struct DevBuf<uint8_t>;
template struct DevBuf<int>;
template struct DevBuf<uint16_t>;
template struct DevBuf<uint32_t>;
template struct DevBuf<unsigned long long>;

// ---- context ---------------------------------------------------------------
Context::Context(int dev) : device(dev) {
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    cuda_check(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
    int major = 0, minor = 0;
    cuda_check(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev), "cc");
    cuda_check(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev), "cc");
    require(major == 10 && minor == 0, "this build targets sm_100a (B200); device is sm_" + std::to_string(major) +
                                           std::to_string(minor));
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    own_stream = true;
}
Context::~Context() {
    if (own_stream && stream) cudaStreamDestroy(stream);
}
void Context::set_stream(cudaStream_t s) {
    if (own_stream && stream) cudaStreamDestroy(stream);
    stream = s;
    own_stream = false;
}

// ---- seeded model init: make_toy_model (ssm.cpp:88-120) with the reference's
// SeededRng (rng.cpp: mt19937_64, explicit Box-Muller with a cached spare).
namespace {
std::vector<double> gaussian(SeededRng& r, size_t n, size_t fan_in) {
    std::vector<double> v(n);
    double s = 1.0 / std::sqrt(static_cast<double>(fan_in));
    for (double& x : v) x = 0.0 + s * r.normal();
    return v;
}
}  // namespace

HostModel make_toy_model(const Dims& d, const std::vector<int>& orders, uint64_t seed) {
    require(d.patch >= 1 && d.image >= d.patch && d.image % d.patch == 0,
            "image side must be a positive multiple of the patch side");
    require(d.channels >= 1 && d.embed >= 1 && d.state >= 1 && d.blocks >= 1 && d.classes >= 2,
            "model dims must be positive (classes >= 2)");
    require(d.conv_width >= 1, "conv width must be >= 1");
    require(!orders.empty() && orders.size() <= 2, "this build supports one or two scan orders");
    for (int o : orders) require(o >= 0 && o <= 3, "unknown scan order value");
    HostModel m;
    m.d = d;
    m.orders = orders;
    SeededRng rng(seed);
    const size_t e = d.embed, n = d.state;
    m.t["patch_w"] = gaussian(rng, e * d.patch_vals(), d.patch_vals());
    m.t["patch_b"] = std::vector<double>(e, 0.0);
    m.t["head_w"] = gaussian(rng, d.classes * e, e);
    m.t["head_b"] = std::vector<double>(d.classes, 0.0);
    for (int b = 0; b < d.blocks; ++b) {
        std::string pb = "block" + std::to_string(b) + ".";
        m.t[pb + "w_in"] = gaussian(rng, e * e, e);
        m.t[pb + "w_gate"] = gaussian(rng, e * e, e);
        m.t[pb + "conv"] = gaussian(rng, e * d.conv_width, d.conv_width);
        m.t[pb + "out_proj"] = gaussian(rng, e * e, e);
        for (size_t k = 0; k < orders.size(); ++k) {
            std::string pd = pb + "dir" + std::to_string(k) + ".";
            std::vector<double> a(e * n);
            for (double& v : a) v = -std::exp(0.0 + (1.0 - 0.0) * rng.uniform());
            m.t[pd + "a"] = a;
            m.t[pd + "w_b"] = gaussian(rng, n * e, e);
            m.t[pd + "w_c"] = gaussian(rng, n * e, e);
            m.t[pd + "w_delta"] = gaussian(rng, e * e, e);
            m.t[pd + "b_delta"] = std::vector<double>(e, 0.0);
        }
    }
    return m;
}

// ---- weight quantization (quantize_weights, quant.cpp:355-372) ----------------
namespace {
double qmax_h(unsigned bits) { return static_cast<double>((1ll << (bits - 1)) - 1); }
struct HostQ {
    std::vector<int8_t> codes;
    std::vector<double> scales, deq;
};
HostQ quantize_rows(const std::vector<double>& w, size_t rows, unsigned bits) {
    HostQ q;
    size_t cols = w.size() / rows;
    double qm = qmax_h(bits);
    q.codes.resize(w.size());
    q.scales.resize(rows);
    q.deq.resize(w.size());
    for (size_t r = 0; r < rows; ++r) {
        const double* row = w.data() + r * cols;
        double mx = 0.0;
        for (size_t c = 0; c < cols; ++c) mx = std::max(mx, std::fabs(row[c]));
        double s = mx == 0.0 ? 1.0 : mx / qm;
        q.scales[r] = s;
        for (size_t c = 0; c < cols; ++c) {
            double v = std::round(row[c] / s);
            if (v > qm) v = qm;
            if (v < -qm) v = -qm;
            q.codes[r * cols + c] = static_cast<int8_t>(v);
        }
    }
    for (size_t i = 0; i < w.size(); ++i) q.deq[i] = static_cast<double>(q.codes[i]) * q.scales[i / cols];
    return q;
}
std::vector<double> cat(std::initializer_list<const std::vector<double>*> parts) {
    std::vector<double> v;
    for (auto* p : parts) v.insert(v.end(), p->begin(), p->end());
    return v;
}
void upload_q(QWeight& qw, const HostQ& q, int rows, int cols, cudaStream_t st) {
    qw.rows = rows;
    qw.cols = cols;
    qw.codes.upload(q.codes.data(), q.codes.size(), st);
    std::vector<int8_t> t(q.codes.size());
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) t[static_cast<size_t>(c) * rows + r] = q.codes[static_cast<size_t>(r) * cols + c];
    qw.codes_t.upload(t.data(), t.size(), st);
    qw.scales.upload(q.scales.data(), q.scales.size(), st);
    cuda_check(cudaStreamSynchronize(st), "upload sync");
}
}  // namespace

Model::Model(Context* c, HostModel hm) : ctx(c), host(std::move(hm)), d(host.d) {}

void Model::set_tensor(const std::string& name, const double* data, size_t n) {
    auto it = host.t.find(name);
    require(it != host.t.end(), "model_set_tensor: unknown tensor '" + name + "'");
    require(it->second.size() == n, "model_set_tensor: size mismatch for '" + name + "'");
    std::memcpy(it->second.data(), data, n * sizeof(double));
    fp_dirty = true;
    qbits = 0;
}

void Model::upload_fp() {
    if (!fp_dirty) return;
    cudaStream_t st = ctx->stream;
    auto& t = host.t;
    patch_w.upload(t["patch_w"].data(), t["patch_w"].size(), st);
    patch_b.upload(t["patch_b"].data(), t["patch_b"].size(), st);
    head_w.upload(t["head_w"].data(), t["head_w"].size(), st);
    head_b.upload(t["head_b"].data(), t["head_b"].size(), st);
    blocks.clear();
    blocks.resize(d.blocks);
    std::vector<std::vector<double>> keep;
    for (int b = 0; b < d.blocks; ++b) {
        std::string pb = "block" + std::to_string(b) + ".";
        keep.push_back(cat({&t[pb + "w_in"], &t[pb + "w_gate"]}));
        blocks[b].w_inproj.upload(keep.back().data(), keep.back().size(), st);
        blocks[b].conv.upload(t[pb + "conv"].data(), t[pb + "conv"].size(), st);
        blocks[b].out_proj.upload(t[pb + "out_proj"].data(), t[pb + "out_proj"].size(), st);
        blocks[b].dirs.resize(host.orders.size());
        for (size_t k = 0; k < host.orders.size(); ++k) {
            std::string pd = pb + "dir" + std::to_string(k) + ".";
            auto& dd = blocks[b].dirs[k];
            dd.a.upload(t[pd + "a"].data(), t[pd + "a"].size(), st);
            dd.b_delta.upload(t[pd + "b_delta"].data(), t[pd + "b_delta"].size(), st);
            keep.push_back(cat({&t[pd + "w_delta"], &t[pd + "w_b"], &t[pd + "w_c"]}));
            dd.xp.upload(keep.back().data(), keep.back().size(), st);
        }
    }
    cuda_check(cudaStreamSynchronize(st), "upload sync");
    fp_dirty = false;
}

std::vector<double> HostModel::dequantized(const std::string& name, unsigned bits) const {
    // quantize_weights + dequantize_rows (quant.cpp:355-384) of one weight matrix; the
    // fused operands are the row concatenations the engine multiplies by
    const int E = d.embed, N = d.state;
    auto at = [&](const std::string& k) -> const std::vector<double>& {
        auto it = t.find(k);
        require(it != t.end(), "qweight: unknown tensor '" + k + "'");
        return it->second;
    };
    const size_t p = name.rfind('.');
    const std::string pre = p == std::string::npos ? "" : name.substr(0, p + 1), leaf = name.substr(p + 1);
    if (name == "patch_w") return quantize_rows(at("patch_w"), E, bits).deq;
    if (name == "head_w") return quantize_rows(at("head_w"), d.classes, bits).deq;
    if (leaf == "in") return quantize_rows(cat({&at(pre + "w_in"), &at(pre + "w_gate")}), 2 * E, bits).deq;
    if (leaf == "out_proj") return quantize_rows(at(name), E, bits).deq;
    if (leaf == "conv") return quantize_rows(at(name), E, bits).deq;
    if (leaf == "xp")
        return quantize_rows(cat({&at(pre + "w_delta"), &at(pre + "w_b"), &at(pre + "w_c")}), E + 2 * N, bits).deq;
    throw ValidationError("qweight: '" + name + "' is not a quantized weight (patch_w, head_w, block<b>.in, "
                          "block<b>.out_proj, block<b>.conv, block<b>.dir<d>.xp)");
}

void Model::quantize(unsigned bits) {
    if (qbits == bits) return;
    upload_fp();
    cudaStream_t st = ctx->stream;
    auto& t = host.t;
    const int E = d.embed, N = d.state;
    HostQ pq = quantize_rows(t["patch_w"], E, bits), hq = quantize_rows(t["head_w"], d.classes, bits);
    patch_deq.upload(pq.deq.data(), pq.deq.size(), st);
    head_deq.upload(hq.deq.data(), hq.deq.size(), st);
    qblocks.clear();
    qblocks.resize(d.blocks);
    for (int b = 0; b < d.blocks; ++b) {
        std::string pb = "block" + std::to_string(b) + ".";
        auto& qb = qblocks[b];
        HostQ in = quantize_rows(cat({&t[pb + "w_in"], &t[pb + "w_gate"]}), 2 * E, bits);
        upload_q(qb.in, in, 2 * E, E, st);
        qb.in_deq.upload(in.deq.data(), in.deq.size(), st);
        HostQ out = quantize_rows(t[pb + "out_proj"], E, bits);
        upload_q(qb.out, out, E, E, st);
        qb.out_deq.upload(out.deq.data(), out.deq.size(), st);
        HostQ cv = quantize_rows(t[pb + "conv"], E, bits);
        qb.conv_deq.upload(cv.deq.data(), cv.deq.size(), st);
        qb.xp.resize(host.orders.size());
        qb.xp_deq.resize(host.orders.size());
        for (size_t k = 0; k < host.orders.size(); ++k) {
            std::string pd = pb + "dir" + std::to_string(k) + ".";
            HostQ xq = quantize_rows(cat({&t[pd + "w_delta"], &t[pd + "w_b"], &t[pd + "w_c"]}), E + 2 * N, bits);
            upload_q(qb.xp[k], xq, E + 2 * N, E, st);
            qb.xp_deq[k].upload(xq.deq.data(), xq.deq.size(), st);
        }
    }
    cuda_check(cudaStreamSynchronize(st), "upload sync");
    qbits = bits;
}

Model::~Model() {
    for (cudaEvent_t e : w.feed_events) cudaEventDestroy(e);
    for (SplitPart& sp : parts) {
        for (cudaEvent_t e : sp.w.feed_events) cudaEventDestroy(e);
        if (sp.fork) cudaEventDestroy(sp.fork);
        if (sp.join) cudaEventDestroy(sp.join);
        if (sp.st) cudaStreamDestroy(sp.st);
        if (sp.copy) cudaStreamDestroy(sp.copy);
    }
}

void Model::ensure_work(Work& w, int S, bool trace) {
    const size_t L = d.tokens(), E = d.embed, N = d.state, nd = host.orders.size();
    const size_t rows = static_cast<size_t>(S) * L;
    w.S = std::max(w.S, S);
    w.x.ensure(rows * E);
    w.patches.ensure(rows * d.patch_vals());
    w.u0.ensure(rows * E);
    w.gate.ensure(rows * E);
    w.u.ensure(rows * E);
    w.xin.ensure(rows * E);
    w.pooled.ensure(static_cast<size_t>(S) * E);
    w.proj.ensure(nd * rows * (E + 2 * N));
    w.o.ensure(nd * rows * E);
    // quantized-activation operands: one slot per scan direction (the x_proj K1 of
    // both directions runs as one launch); slot 0 also serves in_proj / out_proj
    const size_t slots = std::max<size_t>(1, nd);
    w.codes.ensure(slots * rows * E);
    w.codes4.ensure(slots * rows * E / 2);
    w.ocode.ensure(slots * rows * E);
    w.oscale.ensure(slots * rows * E);
    w.omask.ensure(slots * rows * ((E + 31) / 32));
    w.s_row.ensure(slots * rows);
    w.ocnt.ensure(slots * rows);
    w.scanned.ensure(slots * rows);
    w.scan_steps.ensure(scan_fast_workspace_bytes(S, static_cast<int>(L), static_cast<int>(nd), static_cast<int>(E)));
    if (w.merge_cnt.n < static_cast<size_t>(S) * ((E + 31) / 32)) {
        w.merge_cnt.ensure(static_cast<size_t>(S) * ((E + 31) / 32));
        cuda_check(cudaMemset(w.merge_cnt.p, 0, w.merge_cnt.n * sizeof(int)), "merge counters");
    }
    if (trace) {
        w.masks.ensure(2 * 3 * rows * E);
        w.acc_in.ensure(rows * std::max(2 * E, E + 2 * N));
        w.acc_out.ensure(rows * std::max(2 * E, E + 2 * N));
    }
}

// ---- calibration tables -----------------------------------------------------
void Calibration::upload(cudaStream_t st) {
    if (!dirty) return;
    const size_t T = tokens;
    // per tensor: s_in[T] | s_full[T] | 1/s_in[T] | 1/s_full[T]
    std::vector<double> h;
    h.reserve((scan.size() + lin.size()) * 4 * T);
    for (auto* v : {&scan, &lin})
        for (auto& tc : *v) {
            require(tc.s_in.size() == T && tc.s_full.size() == T, "calibration tables have the wrong length");
            h.insert(h.end(), tc.s_in.begin(), tc.s_in.end());
            h.insert(h.end(), tc.s_full.begin(), tc.s_full.end());
            for (double x : tc.s_in) h.push_back(1.0 / x);
            for (double x : tc.s_full) h.push_back(1.0 / x);
        }
    dev.upload(h.data(), h.size(), st);
    // Channel-local detector check C(t) = fl(nextafter(theta,+inf)/q_a) > S^I(t)
    // per scan tensor; a failing step sends that (block, dir)
    // to the literal kernel.
    const double qa = static_cast<double>((1ll << (spec.abits - 1)) - 1);
    std::vector<uint8_t> lit(static_cast<size_t>(blocks) * ndirs * T, 0);
    literal_any.assign(static_cast<size_t>(blocks) * ndirs, 0);
    for (int b = 0; b < blocks; ++b)
        for (int dd = 0; dd < ndirs; ++dd)
            for (int k = 0; k < 3; ++k) {
                const TensorCal& tc = scan[(static_cast<size_t>(b) * ndirs + dd) * 3 + k];
                const double up = std::nextafter(tc.theta, INFINITY) / qa;
                for (size_t t = 0; t < T; ++t)
                    if (!(up > tc.s_in[t])) {
                        lit[(static_cast<size_t>(b) * ndirs + dd) * T + t] = 1;
                        literal_any[static_cast<size_t>(b) * ndirs + dd] = 1;
                    }
            }
    literal.upload(lit.data(), lit.size(), st);
    // the same check for the linear-input sites (K1 channel-parallel kernel)
    lin_literal.assign(lin.size(), 0);
    for (size_t i = 0; i < lin.size(); ++i) {
        const double up = std::nextafter(lin[i].theta, INFINITY) / qa;
        for (size_t t = 0; t < T; ++t)
            if (!(up > lin[i].s_in[t])) lin_literal[i] = 1;
    }
    cuda_check(cudaStreamSynchronize(st), "calib upload");
    dirty = false;
}
const double* Calibration::s_in_dev(bool is_lin, size_t idx) const {
    size_t base = (is_lin ? scan.size() + idx : idx) * 4 * tokens;
    return dev.p + base;
}
const double* Calibration::s_full_dev(bool is_lin, size_t idx) const { return s_in_dev(is_lin, idx) + tokens; }
const double* Calibration::inv_in_dev(bool is_lin, size_t idx) const { return s_in_dev(is_lin, idx) + 2 * tokens; }
const double* Calibration::inv_full_dev(bool is_lin, size_t idx) const { return s_in_dev(is_lin, idx) + 3 * tokens; }

// ---- forward ------------------------------------------------------------------
namespace {
template <class T>
void grab(Model::TraceSink* tr, const std::string& key, const T* dev, size_t n, cudaStream_t st) {
    std::vector<char> b(n * sizeof(T));
    cuda_check(cudaStreamSynchronize(st), "trace sync");
    cuda_check(cudaMemcpy(b.data(), dev, b.size(), cudaMemcpyDeviceToHost), "trace copy");
    tr->blobs[key] = std::move(b);
}
}  // namespace

void Model::forward(const Calibration* cal, int mode, bool d1, bool d2, const double* images, int S, double* logits,
                    TraceSink* trace, unsigned long long* calib_peaks, const HostFeed* feed) {
    require(S >= 1, "forward: batch must be >= 1");
    require(d.state == 16, "this build keeps N = 16 scan states in registers (ModelDims.state must be 16)");
    require(d.embed % 32 == 0 && d.embed <= 1024, "embed must be a multiple of 32 and <= 1024");
    const bool quant = mode != MODE_FP;
    if (quant) {
        require(cal != nullptr, "quantized modes need a calibration");
        require(cal->blocks == d.blocks && cal->ndirs == static_cast<int>(host.orders.size()) &&
                    cal->tokens == d.tokens() && cal->embed == d.embed,
                "calibration does not match the model geometry");  // quant.cpp:508-510
        if (d2) require(cal->d2 && cal->lin.size() == static_cast<size_t>(cal->blocks) * cal->nsites(),
                        "calibration lacks linear-input records (D2)");
        // thresholds and scales were recorded on the D1 (pre-norm) or the raw
        // activation distribution; the other one would be silently miscalibrated
        require(cal->d1 == d1, "calibration was recorded with d1 = " + std::to_string(cal->d1 ? 1 : 0) +
                                   " but the forward runs with d1 = " + std::to_string(d1 ? 1 : 0));
        quantize(cal->spec.wbits);
        const_cast<Calibration*>(cal)->upload(ctx->stream);
    }
    upload_fp();
    const int np = std::min(split_parts, kMaxSplit);
    const bool split = np > 1 && trace == nullptr && calib_peaks == nullptr && !timing.on && S >= np * kSplitMin &&
                       static_cast<long>(S) * d.tokens() >= static_cast<long>(np) * split_min_rows;
    if (!split) {
        forward_impl(cal, mode, d1, d2, images, S, logits, trace, calib_peaks, feed, ctx->stream, w);
        return;
    }
    const size_t pix = static_cast<size_t>(d.image) * d.image * d.channels;
    for (int k = 1; k < np; ++k) {
        SplitPart& sp = parts[k];
        if (sp.st == nullptr) {
            cuda_check(cudaStreamCreateWithFlags(&sp.st, cudaStreamNonBlocking), "split stream");
            cuda_check(cudaStreamCreateWithFlags(&sp.copy, cudaStreamNonBlocking), "split copy stream");
            cuda_check(cudaEventCreateWithFlags(&sp.fork, cudaEventDisableTiming), "split event");
            cuda_check(cudaEventCreateWithFlags(&sp.join, cudaEventDisableTiming), "split event");
        }
        cuda_check(cudaEventRecord(sp.fork, ctx->stream), "split fork");
        cuda_check(cudaStreamWaitEvent(sp.st, sp.fork, 0), "split fork");
    }
    for (int k = 0; k < np; ++k) {
        const int s0 = static_cast<int>(static_cast<long>(S) * k / np);
        const int s1 = static_cast<int>(static_cast<long>(S) * (k + 1) / np);
        HostFeed f;
        if (feed) {
            f = *feed;
            f.chunks = std::max(1, feed->chunks / np);
            f.host = feed->host + static_cast<size_t>(s0) * pix;
            if (k > 0) f.copy = parts[k].copy;  // every part's first chunk arrives early (they share PCIe)
        }
        forward_impl(cal, mode, d1, d2, images + static_cast<size_t>(s0) * pix, s1 - s0,
                     logits + static_cast<size_t>(s0) * d.classes, nullptr, nullptr, feed ? &f : nullptr,
                     k == 0 ? ctx->stream : parts[k].st, k == 0 ? w : parts[k].w, s0);
    }
    for (int k = 1; k < np; ++k) {
        cuda_check(cudaEventRecord(parts[k].join, parts[k].st), "split join");
        cuda_check(cudaStreamWaitEvent(ctx->stream, parts[k].join, 0), "split join");
    }
}

void Model::forward_impl(const Calibration* cal, int mode, bool d1, bool d2, const double* images, int S,
                         double* logits, TraceSink* trace, unsigned long long* calib_peaks, const HostFeed* feed,
                         cudaStream_t st, Work& w, int sample0) {
    const bool quant = mode != MODE_FP;
    const bool qlin = quant && d2;
    ensure_work(w, S, trace != nullptr);
    const int L = d.tokens(), E = d.embed, N = d.state, nd = static_cast<int>(host.orders.size());
    const int P = E + 2 * N, nsites = nd + 2;
    const size_t rows = static_cast<size_t>(S) * L;
    const bool tr_on = trace != nullptr;
    auto tb = [&](int b) { return tr_on && trace->block == b; };

    // patch embed: x = patches . W^T + b (ssm.cpp:253-256), FP or W4-dequantized weights;
    // per-sample work, so with a host feed it runs chunk by chunk behind the H2D copies
    const size_t pix = static_cast<size_t>(d.image) * d.image * d.channels;
    const int nchunk = feed ? std::max(1, std::min(feed->chunks, S)) : 1;
    if (feed) {
        auto& feed_events = w.feed_events;
        while (static_cast<int>(feed_events.size()) < nchunk + 1) {
            cudaEvent_t e;
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            feed_events.push_back(e);
        }
        cuda_check(cudaEventRecord(feed_events[nchunk], st), "feed fork");  // copies start after prior work
        cuda_check(cudaStreamWaitEvent(feed->copy, feed_events[nchunk], 0), "feed fork");
        for (int k = 0; k < nchunk; ++k) {
            const int s0 = static_cast<int>(static_cast<long>(S) * k / nchunk);
            const int s1 = static_cast<int>(static_cast<long>(S) * (k + 1) / nchunk);
            cuda_check(cudaMemcpyAsync(const_cast<double*>(images) + s0 * pix, feed->host + s0 * pix,
                                       (s1 - s0) * pix * sizeof(double), cudaMemcpyHostToDevice, feed->copy),
                       "H2D images");
            cuda_check(cudaEventRecord(w.feed_events[k], feed->copy), "feed event");
        }
    }
    for (int k = 0; k < nchunk; ++k) {
        const int s0 = static_cast<int>(static_cast<long>(S) * k / nchunk);
        const int s1 = static_cast<int>(static_cast<long>(S) * (k + 1) / nchunk);
        if (feed) cuda_check(cudaStreamWaitEvent(st, w.feed_events[k], 0), "feed wait");
        const size_t r0 = static_cast<size_t>(s0) * L, nr = static_cast<size_t>(s1 - s0) * L;
        tick_begin(FAM_AUX);
        cuda_check(launch_patch_gather(images + s0 * pix, w.patches.p + r0 * d.patch_vals(), s1 - s0, d.image,
                                       d.channels, d.patch, st),
                   "patch gather");
        tick_end(FAM_AUX);
        DGemmParams g;
        g.M = static_cast<int>(nr);
        g.R = E;
        g.K = d.patch_vals();
        g.a = w.patches.p + r0 * d.patch_vals();
        g.lda = d.patch_vals();
        g.w = quant ? patch_deq.p : patch_w.p;
        g.epi.post = POST_BIAS;
        g.epi.out = w.x.p + r0 * E;
        g.epi.ld_out = E;
        g.epi.bias = patch_b.p;
        tick_begin(FAM_DGEMM);
        cuda_check(launch_dgemm(g, st), "patch embed");
        tick_end(FAM_DGEMM);
    }
    if (tr_on) grab(trace, "x_embed", w.x.p, rows * E, st);

    int qslot = 0;  // QAct slot the K1 / K2 / trace lambdas address
    const size_t J = (E + 31) / 32;
    const bool pk = qlin && pack_a4 && cal->spec.abits == 4;  // nibble-packed A4 operand
    auto k1_base = [&](int src, const double* x, int order, int b, int site, bool record) {
        K1Params k;
        k.S = S;
        k.T = L;
        k.E = E;
        k.src = src;
        k.x = x;
        k.order = order;
        k.grid = d.grid();
        if (qlin) {
            const size_t li = static_cast<size_t>(b) * nsites + site;
            k.mode = mode;
            k.n_refresh = cal->spec.n_refresh;
            k.abits = cal->spec.abits;
            k.obits = cal->spec.obits;
            k.window = (mode == MODE_DYNAMIC) ? (cal->spec.n_refresh > 0 ? cal->spec.n_refresh : L) : 8;
            k.cal.theta = cal->lin[li].theta;
            k.cal.s_in = cal->s_in_dev(true, li);
            k.cal.s_full = cal->s_full_dev(true, li);
            k.inv_in = cal->inv_in_dev(true, li);
            k.inv_full = cal->inv_full_dev(true, li);
            if (pk) k.codes4 = w.codes4.p + qslot * rows * E / 2;
            else k.codes = w.codes.p + qslot * rows * E;
            k.s_row = w.s_row.p + qslot * rows;
            k.ocnt = w.ocnt.p + qslot * rows;
            k.omask = w.omask.p + qslot * rows * J;
            k.ocode = w.ocode.p + qslot * rows * E;
            k.oscale = w.oscale.p + qslot * rows * E;
            // literal detector where the channel-local form is not exact, on request,
            // and in trace mode (it also reports DetectResult::scanned)
            k.force_literal = (mode == MODE_DYNAMIC && cal->lin_literal[li]) || k1_variant == 1 || tb(b);
            k.window_kernel = k1_variant == 2;
            if (tb(b)) k.scanned = w.scanned.p + qslot * rows;
        } else {
            k.mode = MODE_FP;
            k.window = 8;
            k.xout = w.xin.p;
            if (record && calib_peaks) k.peaks = calib_peaks + (static_cast<size_t>(b) * nsites + site) * L * E;
        }
        return k;
    };
    auto qact = [&]() {
        QAct a;
        if (pk) a.codes4 = w.codes4.p + qslot * rows * E / 2;
        else a.codes = w.codes.p + qslot * rows * E;
        a.s_row = w.s_row.p + qslot * rows;
        a.ocnt = w.ocnt.p + qslot * rows;
        a.omask = w.omask.p + qslot * rows * J;
        a.ocode = w.ocode.p + qslot * rows * E;
        a.oscale = w.oscale.p + qslot * rows * E;
        a.J = static_cast<int>(J);
        return a;
    };
    auto trace_lin = [&](int b, int site, int R) {
        if (!tb(b) || !qlin) return;
        std::string p = "lin" + std::to_string(site) + ".";
        if (pk) {  // the packed operand, and its codes unpacked (one int8 per code) for the parity checks
            grab(trace, p + "codes4", w.codes4.p + qslot * rows * E / 2, rows * E / 2, st);
            const std::vector<char>& b4 = trace->blobs[p + "codes4"];
            std::vector<char> c(rows * E);
            unpack_nibbles(reinterpret_cast<const uint8_t*>(b4.data()), rows * E, reinterpret_cast<int8_t*>(c.data()));
            trace->blobs[p + "codes"] = std::move(c);
        } else {
            grab(trace, p + "codes", w.codes.p + qslot * rows * E, rows * E, st);
        }
        grab(trace, p + "s_row", w.s_row.p + qslot * rows, rows, st);
        grab(trace, p + "ocnt", w.ocnt.p + qslot * rows, rows, st);
        grab(trace, p + "ocode", w.ocode.p + qslot * rows * E, rows * E, st);
        grab(trace, p + "oscale", w.oscale.p + qslot * rows * E, rows * E, st);
        grab(trace, p + "omask", w.omask.p + qslot * rows * J, rows * J, st);
        grab(trace, p + "scanned", w.scanned.p + qslot * rows, rows, st);
        grab(trace, p + "acc_in", w.acc_in.p, rows * R, st);
        grab(trace, p + "acc_out", w.acc_out.p, rows * R, st);
    };
    auto linear = [&](const QWeight* qw, const double* wdeq_or_fp, int R, const GemmEpi& epi_in, int b) {
        GemmEpi epi = epi_in;
        if (qlin) {
            if (tb(b)) {
                epi.acc_in = w.acc_in.p;
                epi.acc_out = w.acc_out.p;
            }
            QLinParams q;
            q.M = static_cast<int>(rows);
            q.R = R;
            q.K = E;
            q.a = qact();
            q.w = qw->codes.p;
            q.wt = qw->codes_t.p;
            q.ws = qw->scales.p;
            q.epi = epi;
            tick_begin(FAM_K2);
            cuda_check(launch_qlinear(q, st, ctx->num_sms), "quant linear");
            tick_end(FAM_K2);
        } else {
            DGemmParams g;
            g.M = static_cast<int>(rows);
            g.R = R;
            g.K = E;
            g.a = w.xin.p;
            g.lda = E;
            g.w = wdeq_or_fp;
            g.epi = epi;
            tick_begin(FAM_DGEMM);
            cuda_check(launch_dgemm(g, st), "f64 linear");
            tick_end(FAM_DGEMM);
        }
    };

    for (int b = 0; b < d.blocks; ++b) {
        const BlockDev& bd = blocks[b];
        const BlockQ* bq = quant ? &qblocks[b] : nullptr;
        if (tb(b)) grab(trace, "x_in", w.x.p, rows * E, st);
        // in_proj input: RMSNorm(x) (D1) or x
        K1Params k = k1_base(d1 ? K1_SRC_RMSNORM : K1_SRC_PLAIN, w.x.p, -1, b, 0, true);
        tick_begin(FAM_K1);
        cuda_check(launch_k1(k, st), "K1 in_proj");
        tick_end(FAM_K1);
        if (tb(b) && !qlin) grab(trace, "xn", w.xin.p, rows * E, st);
        {
            GemmEpi e;
            e.post = POST_INPROJ;
            e.out = w.u0.p;
            e.ld_out = E;
            e.out2 = w.gate.p;
            e.split = E;
            linear(bq ? &bq->in : nullptr, quant ? bq->in_deq.p : bd.w_inproj.p, 2 * E, e, b);
            trace_lin(b, 0, 2 * E);
        }
        tick_begin(FAM_AUX);
        cuda_check(launch_conv(w.u0.p, quant ? bq->conv_deq.p : bd.conv.p, w.u.p, S, L, E, d.conv_width, st), "conv");
        tick_end(FAM_AUX);
        if (tb(b)) {
            grab(trace, "u0", w.u0.p, rows * E, st);
            grab(trace, "gate_pre", w.gate.p, rows * E, st);
            grab(trace, "u", w.u.p, rows * E, st);
        }
        ScanParams sps[2];
        bool any_literal = false;
        // x_proj inputs of every direction: one K1 launch over the shared rows u
        // (direction dd quantizes into QAct slot dd), then the x_proj GEMMs. FP mode
        // materialises rows into the one xin buffer: K1 and GEMM per direction.
        const bool k1_pair = qlin && nd <= 2;
        if (k1_pair) {
            K1Params kx[2];
            for (int dd = 0; dd < nd; ++dd) {
                qslot = dd;
                kx[dd] = k1_base(K1_SRC_PLAIN, w.u.p, host.orders[dd], b, 1 + dd, true);
            }
            tick_begin(FAM_K1);
            cuda_check(launch_k1_dirs(kx, nd, st), "K1 x_proj");
            tick_end(FAM_K1);
        }
        for (int dd = 0; dd < nd; ++dd) {
            const int order = host.orders[dd];
            double* proj = w.proj.p + static_cast<size_t>(dd) * rows * P;
            double* o = w.o.p + static_cast<size_t>(dd) * rows * E;
            qslot = k1_pair ? dd : 0;
            if (!k1_pair) {
                K1Params kx = k1_base(K1_SRC_PLAIN, w.u.p, order, b, 1 + dd, true);
                tick_begin(FAM_K1);
                cuda_check(launch_k1(kx, st), "K1 x_proj");
                tick_end(FAM_K1);
            }
            GemmEpi e;  // dpre | B | C (softplus(dpre + b_delta) runs in the scan's chunk pre-pass)
            e.post = POST_STORE;
            e.out = proj;
            e.ld_out = P;
            linear(bq ? &bq->xp[dd] : nullptr, quant ? bq->xp_deq[dd].p : bd.dirs[dd].xp.p, P, e, b);
            trace_lin(b, 1 + dd, P);
            ScanParams& sp = sps[dd];
            sp = ScanParams{};
            sp.S = S;
            sp.T = L;
            sp.E = E;
            sp.N = N;
            sp.order = order;
            sp.grid = d.grid();
            sp.u = w.u.p;
            sp.proj = proj;
            sp.a = bd.dirs[dd].a.p;
            sp.b_delta = bd.dirs[dd].b_delta.p;
            sp.o = o;
            sp.mode = mode;
            if (quant) {
                sp.n_refresh = cal->spec.n_refresh;
                sp.abits = cal->spec.abits;
                sp.obits = cal->spec.obits;
                for (int kk = 0; kk < 3; ++kk) {
                    const size_t si = (static_cast<size_t>(b) * nd + dd) * 3 + kk;
                    sp.cal[kk].theta = cal->scan[si].theta;
                    sp.cal[kk].s_in = cal->s_in_dev(false, si);
                    sp.cal[kk].s_full = cal->s_full_dev(false, si);
                    sp.cal[kk].inv_in = cal->inv_in_dev(false, si);
                    sp.cal[kk].inv_full = cal->inv_full_dev(false, si);
                }
                sp.literal = cal->literal.p + (static_cast<size_t>(b) * nd + dd) * L;
                sp.literal_any = mode == MODE_DYNAMIC ? cal->literal_any[static_cast<size_t>(b) * nd + dd] : 0;
                any_literal = any_literal || sp.literal_any;
                if (tb(b)) sp.masks = w.masks.p + static_cast<size_t>(dd) * 3 * rows * E;
            } else if (calib_peaks) {
                const size_t base = static_cast<size_t>(d.blocks) * nsites * L * E;
                for (int kk = 0; kk < 3; ++kk)
                    sp.cal[kk].peaks = calib_peaks + base + ((static_cast<size_t>(b) * nd + dd) * 3 + kk) * L * E;
            }
        }
        // K3: both directions in one launch on the fast path; the literal
        // detector (or FP recording) runs the per-direction kernel.
        bool lit = false;
        tick_begin(FAM_K3);
        const bool fast_ok = quant && cal->spec.obits == 8 && (cal->spec.abits == 4 || cal->spec.abits == 8);
        for (int dd = 0; dd < nd; ++dd) {  // SpikeHook runs in the reference-form kernel
            sps[dd].spike = spikes;
            sps[dd].spike.block = b;
            sps[dd].spike.dir = dd;
            sps[dd].spike.sample0 = spikes.sample0 + sample0;
        }
        // the out_proj input K1 (merge source) rides on the fast scan's tail where that
        // kernel runs it (qslot 0, its |O(t)| zeroed first); else it runs after the scan
        qslot = 0;
        K1Params km = k1_base(K1_SRC_MERGE, w.o.p, -1, b, nsites - 1, true);
        km.x2 = nd > 1 ? w.o.p + rows * E : nullptr;
        km.gate = w.gate.p;
        bool merged = false;
        if (fast_ok && !any_literal && scan_variant != 1 && !(spikes.rate > 0.0)) {
            const bool fuse = qlin && merge_fuse && !km.force_literal && !km.scanned;
            if (fuse) cuda_check(cudaMemsetAsync(km.ocnt, 0, rows * sizeof(int), st), "merge ocnt");
            cuda_check(launch_scan_fast(sps, nd, w.scan_steps.p, w.scan_steps.n, st, scan_variant >= 2 ? scan_variant - 1 : 0,
                                        fuse ? &km : nullptr, fuse ? w.merge_cnt.p : nullptr, &merged),
                       "scan");
        } else {
            for (int dd = 0; dd < nd; ++dd) {
                bool l = false;
                cuda_check(launch_scan(sps[dd], st, &l), "scan");
                lit = lit || l;
            }
        }
        tick_end(FAM_K3);
        if (tb(b))
            for (int dd = 0; dd < nd; ++dd) {
                std::string p = "dir" + std::to_string(dd) + ".";
                grab(trace, p + "proj", sps[dd].proj, rows * P, st);
                grab(trace, p + "o", sps[dd].o, rows * E, st);
                if (quant && mode == MODE_DYNAMIC) grab(trace, p + "masks", sps[dd].masks, 3 * rows * E, st);
                trace->blobs[p + "literal"] = std::vector<char>(1, static_cast<char>(lit ? 1 : 0));
            }
        if (!merged) {
            tick_begin(FAM_K1);
            cuda_check(launch_k1(km, st), "K1 out_proj");
            tick_end(FAM_K1);
        }
        if (tb(b) && !qlin) grab(trace, "y", w.xin.p, rows * E, st);
        {
            GemmEpi e;
            e.post = d1 ? POST_RESID : POST_STORE;
            e.out = w.x.p;
            e.ld_out = E;
            linear(bq ? &bq->out : nullptr, quant ? bq->out_deq.p : bd.out_proj.p, E, e, b);
            trace_lin(b, nsites - 1, E);
        }
        if (tb(b)) grab(trace, "x_out", w.x.p, rows * E, st);
    }
    tick_begin(FAM_AUX);
    cuda_check(launch_meanpool(w.x.p, w.pooled.p, S, L, E, st), "meanpool");
    tick_end(FAM_AUX);
    {
        DGemmParams g;
        g.M = S;
        g.R = d.classes;
        g.K = E;
        g.a = w.pooled.p;
        g.lda = E;
        g.w = quant ? head_deq.p : head_w.p;
        g.epi.post = POST_BIAS;
        g.epi.out = logits;
        g.epi.ld_out = d.classes;
        g.epi.bias = head_b.p;
        tick_begin(FAM_DGEMM);
        cuda_check(launch_dgemm(g, st), "head");
        tick_end(FAM_DGEMM);
    }
}

void Model::tick_begin(int fam) {
    if (!timing.on) return;
    cudaEvent_t a, b;
    cuda_check(cudaEventCreate(&a), "event");
    cuda_check(cudaEventCreate(&b), "event");
    cuda_check(cudaEventRecord(a, ctx->stream), "event record");
    timing.ev.push_back({fam, {a, b}});
    timing.k0 = kernel_launch_counter();
}
void Model::tick_end(int fam) {
    if (!timing.on) return;
    cuda_check(cudaEventRecord(timing.ev.back().second.second, ctx->stream), "event record");
    timing.launches[fam] += static_cast<int>(kernel_launch_counter() - timing.k0);  // kernels, not ops
}
void Model::timing_collect() {
    cuda_check(cudaStreamSynchronize(ctx->stream), "timing sync");
    for (auto& e : timing.ev) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, e.second.first, e.second.second), "elapsed");
        timing.ms[e.first] += ms;
        if (timing.keep_list) timing.list.push_back({e.first, static_cast<double>(ms)});
        cudaEventDestroy(e.second.first);
        cudaEventDestroy(e.second.second);
    }
    timing.ev.clear();
}

// calibrate (quant.cpp:129-177) on the device: FP forward with per-(tensor, t,
// ch) peak recording (atomicMax over samples), then the quantile reduction on
// the host.
std::unique_ptr<Calibration> Model::calibrate(const double* images_dev, int S, const QuantSpec& spec, bool d1,
                                              bool d2, int chunk) {
    spec.validate();
    const int L = d.tokens(), E = d.embed, nd = static_cast<int>(host.orders.size());
    const size_t nlin = d2 ? static_cast<size_t>(d.blocks) * (nd + 2) : 0;
    const size_t nscan = static_cast<size_t>(d.blocks) * nd * 3;
    const size_t nsites_total = static_cast<size_t>(d.blocks) * (nd + 2);
    DevBuf<unsigned long long> peaks;
    peaks.ensure((nsites_total + nscan) * L * E);
    cuda_check(cudaMemsetAsync(peaks.p, 0, peaks.n * sizeof(unsigned long long), ctx->stream), "memset");
    DevBuf<double> logits;
    const int ch = chunk > 0 ? std::min(chunk, S) : S;
    logits.ensure(static_cast<size_t>(ch) * d.classes);
    const size_t pix = static_cast<size_t>(d.image) * d.image * d.channels;
    for (int s0 = 0; s0 < S; s0 += ch) {
        const int n = std::min(ch, S - s0);
        forward(nullptr, MODE_FP, d1, d2, images_dev + s0 * pix, n, logits.p, nullptr, peaks.p);
    }
    std::vector<unsigned long long> h(peaks.n);
    cuda_check(cudaStreamSynchronize(ctx->stream), "calibrate");
    cuda_check(cudaMemcpy(h.data(), peaks.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "d2h");
    auto cal = std::make_unique<Calibration>();
    cal->spec = spec;
    cal->d1 = d1;
    cal->d2 = d2;
    cal->tokens = L;
    cal->embed = E;
    cal->blocks = d.blocks;
    cal->ndirs = nd;
    const double qa = qmax_h(spec.abits);
    auto reduce = [&](const unsigned long long* pk) {  // quant.cpp:145-176
        TensorCal tc;
        std::vector<double> peak(static_cast<size_t>(L) * E);
        for (size_t i = 0; i < peak.size(); ++i) std::memcpy(&peak[i], &pk[i], sizeof(double));
        std::vector<double> pooled(E, 0.0);
        for (int t = 0; t < L; ++t)
            for (int c = 0; c < E; ++c) pooled[c] = std::max(pooled[c], peak[static_cast<size_t>(t) * E + c]);
        std::vector<double> v = pooled;  // quantile, quant.cpp:117-125
        std::sort(v.begin(), v.end());
        double pos = (1.0 - spec.rho) * static_cast<double>(v.size() - 1);
        size_t lo = static_cast<size_t>(pos);
        tc.theta = lo + 1 >= v.size() ? v.back() : v[lo] + (pos - static_cast<double>(lo)) * (v[lo + 1] - v[lo]);
        tc.excluded.resize(E);
        for (int c = 0; c < E; ++c) tc.excluded[c] = pooled[c] > tc.theta ? 1 : 0;
        tc.s_in.resize(L);
        tc.s_full.resize(L);
        for (int t = 0; t < L; ++t) {
            double mi = 0.0, mf = 0.0;
            for (int c = 0; c < E; ++c) {
                double p = peak[static_cast<size_t>(t) * E + c];
                mf = std::max(mf, p);
                if (!tc.excluded[c]) mi = std::max(mi, p);
            }
            tc.s_in[t] = mi == 0.0 ? 1.0 : mi / qa;
            tc.s_full[t] = mf == 0.0 ? 1.0 : mf / qa;
        }
        return tc;
    };
    const unsigned long long* scanp = h.data() + nsites_total * L * E;
    for (size_t i = 0; i < nscan; ++i) cal->scan.push_back(reduce(scanp + i * L * E));
    for (size_t i = 0; i < nlin; ++i) cal->lin.push_back(reduce(h.data() + i * L * E));
    return cal;
}

}  // namespace ob
