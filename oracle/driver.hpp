// ORACLE — test infrastructure only. Never linked into the product.
//
// Model-level driver of the OuroMamba-Quant Vim forward, shared by the two CPU
// checkers of this repo:
//   * liboracle.so        Driver<OracleOps>  (oracle/oracle_ops.hpp restatement)
//   * _ref/libouro_ref.so Driver<RefOps>     (the reference's own compiled
//                                             functions, oracle/ref/ref_ops.hpp)
// The driver restates the parts of the reference that live in anonymous
// namespaces and cannot be called: the block (ssm.cpp:192-233), the per-step
// quantization policy QuantHook (quant.cpp:456-501), the calibration recorder
// (quant.cpp:82-114) and calibrate's reduction (quant.cpp:129-177). With both
// extensions off, Driver<RefOps> is pinned bit-for-bit against the reference's
// exported vmm_forward_raw / quantized_forward / calibrate.
//
// Declared extensions:
//   D1 pre-norm residual: x <- x + Block(RMSNorm(x)), RMSNorm(x) = x * (1/sqrt(ms+1e-6)),
//      ms = sum(x^2)/E with the sum taken as 32 lane-strided partials (channel
//      k goes to partial k%32, k ascending) combined by an xor-butterfly
//      (offsets 16,8,4,2,1) — the order a warp computes it in.
//   D2 linear-input quantization: the inputs of in_proj, x_proj/dt_proj (per
//      dir) and out_proj go through maybe_refresh -> detect_outliers ->
//      split_quantize -> hybrid_gemm, one (sample, token) plane (K=E channels,
//      C=1 column) per step; the outlier state is carried along the token
//      order of the layer (canonical for in/out_proj, scan order for x_proj)
//      and refreshed every n_refresh tokens, exactly like the scan tensors.
#pragma once
#include <cstring>
#include <memory>
#include <thread>

#include "oracle_ops.hpp"

namespace oro {

struct Spec {  // QuantSpec, quant.hpp:21-28
    unsigned wbits = 4, abits = 8, obits = 8;
    std::size_t n_refresh = 10;
    double rho = 0.01;
    void validate() const {  // quant.cpp:54-60
        require(wbits >= 2, "weight bits must be >= 2");
        require(abits >= 2, "activation bits must be >= 2");
        require(obits >= 2 && obits <= 8, "outlier bits must be in [2, 8]");
        require(abits <= obits, "inlier activation bits must not exceed outlier bits");
        require(rho >= 0.0 && rho < 1.0, "rho must be in [0, 1)");
    }
};
struct TCal {  // TensorCalib, quant.hpp:36-42
    double theta = 0.0;
    std::vector<double> s_in, s_full;
    std::vector<char> excluded;
};
enum Kind { ABAR = 0, BBAR = 1, HST = 2 };  // ActKind, quant.hpp:32
struct Calib {
    Spec spec;
    std::size_t tokens = 0, embed = 0, state = 0, blocks = 0, ndirs = 0;
    bool d1 = true, d2 = true;
    std::vector<TCal> scan;  // [block][dir][kind], quant.cpp:71-75
    std::vector<TCal> lin;   // [block][site], site 0 in_proj, 1..ndirs x_proj dir, ndirs+1 out_proj
    std::size_t nsites() const { return ndirs + 2; }
    const TCal& at(std::size_t b, std::size_t d, int k) const { return scan[(b * ndirs + d) * 3 + k]; }
    const TCal& site(std::size_t b, std::size_t s) const { return lin[b * nsites() + s]; }
};
enum Mode { MODE_FP = 0, MODE_DYNAMIC = 1, MODE_STATIC = 2 };

// Per-(tensor, t, ch) peaks pooled over samples: CalibRecorder, quant.cpp:82-114.
struct Recorder {
    std::size_t tokens, embed;
    std::vector<std::vector<double>> scan, lin;  // peak[t*E + ch]
    Recorder(std::size_t L, std::size_t E, std::size_t nscan, std::size_t nlin)
        : tokens(L), embed(E), scan(nscan, std::vector<double>(L * E, 0.0)),
          lin(nlin, std::vector<double>(L * E, 0.0)) {}
    static void note(std::vector<double>& peaks, std::size_t t, const double* x, std::size_t e,
                     std::size_t n) {
        for (std::size_t ch = 0; ch < e; ++ch) {
            double mx = 0.0;
            for (std::size_t s = 0; s < n; ++s) mx = std::max(mx, std::fabs(x[ch * n + s]));
            double& p = peaks[t * e + ch];
            p = std::max(p, mx);
        }
    }
    void merge(const Recorder& o) {
        for (std::size_t i = 0; i < scan.size(); ++i)
            for (std::size_t j = 0; j < scan[i].size(); ++j) scan[i][j] = std::max(scan[i][j], o.scan[i][j]);
        for (std::size_t i = 0; i < lin.size(); ++i)
            for (std::size_t j = 0; j < lin[i].size(); ++j) lin[i][j] = std::max(lin[i][j], o.lin[i][j]);
    }
};

// Reduction of calibrate(), quant.cpp:145-176, for one tensor's peaks.
inline TCal reduce_calib(const std::vector<double>& peaks, std::size_t L, std::size_t E, double rho,
                         unsigned abits) {
    double qa = qmax_for(abits);
    TCal tc;
    std::vector<double> pooled(E, 0.0);
    for (std::size_t t = 0; t < L; ++t)
        for (std::size_t ch = 0; ch < E; ++ch) pooled[ch] = std::max(pooled[ch], peaks[t * E + ch]);
    tc.theta = quantile(pooled, 1.0 - rho);
    tc.excluded.resize(E);
    for (std::size_t ch = 0; ch < E; ++ch) tc.excluded[ch] = pooled[ch] > tc.theta ? 1 : 0;
    tc.s_in.resize(L);
    tc.s_full.resize(L);
    for (std::size_t t = 0; t < L; ++t) {
        double mi = 0.0, mf = 0.0;
        for (std::size_t ch = 0; ch < E; ++ch) {
            double p = peaks[t * E + ch];
            mf = std::max(mf, p);
            if (!tc.excluded[ch]) mi = std::max(mi, p);
        }
        tc.s_in[t] = mi == 0.0 ? 1.0 : mi / qa;
        tc.s_full[t] = mf == 0.0 ? 1.0 : mf / qa;
    }
    return tc;
}

// D1 RMSNorm of one token row (order documented in the header).
inline void rmsnorm_row(const double* x, double* y, std::size_t e) {
    double p[32];
    for (int l = 0; l < 32; ++l) {
        double s = 0.0;
        for (std::size_t k = static_cast<std::size_t>(l); k < e; k += 32) s = s + x[k] * x[k];
        p[l] = s;
    }
    for (int off = 16; off >= 1; off >>= 1) {
        double q[32];
        for (int l = 0; l < 32; ++l) q[l] = p[l] + p[l ^ off];
        std::memcpy(p, q, sizeof p);
    }
    double ms = p[0] / static_cast<double>(e);
    double r = 1.0 / std::sqrt(ms + 1e-6);
    for (std::size_t k = 0; k < e; ++k) y[k] = x[k] * r;
}

// Everything one block computed for one sample (captured on request).
struct LinTrace {
    std::vector<std::int8_t> codes, ocode;  // L x E (inlier codes, 0 at outliers) / outlier codes
    std::vector<std::uint8_t> omask;        // L x E, O(t) after detection
    std::vector<double> oscale;             // L x E, per-channel outlier scale at O(t)
    std::vector<std::int32_t> acc_in, acc_out;  // L x R
    std::vector<double> out;                    // L x R
    std::vector<std::uint8_t> scanned;          // L
};
struct DirTrace {
    std::vector<double> u, delta, o;                 // L x E, scan order
    std::vector<double> bvec, cvec;                  // L x N
    std::vector<std::uint8_t> mask[3];               // L x E, O(t) per kind after detection
    std::vector<std::uint8_t> scanned[3];            // L
};
struct BlockTrace {
    std::vector<double> x_in, xn, u0, gate, gpre, u, merged, y, x_out;  // L x E
    LinTrace lin[6];                                              // sites (ndirs <= 4)
    std::vector<DirTrace> dirs;
};

struct QModel {  // quantize_model_weights, quant.cpp:384-402, plus the D2 operand view
    QRows patch, head;
    struct Blk {
        QRows in, conv, out;  // in: 2E rows (w_in then w_gate)
        std::vector<QRows> xp;  // per dir: E+2N rows (w_delta, w_b, w_c)
    };
    std::vector<Blk> blocks;
};
template <class Ops>
QModel quantize_model(const ModelW& m, unsigned bits) {
    QModel q;
    std::size_t e = m.d.embed, n = m.d.state;
    auto quantize_rows = [](const std::vector<double>& w, std::size_t rows, unsigned b) {
        return Ops::quantize_rows(w, rows, b);
    };
    q.patch = quantize_rows(m.patch_w, e, bits);
    q.head = quantize_rows(m.head_w, m.d.classes, bits);
    for (const BlockW& b : m.blocks) {
        QModel::Blk qb;
        std::vector<double> in(b.w_in);
        in.insert(in.end(), b.w_gate.begin(), b.w_gate.end());
        qb.in = quantize_rows(in, 2 * e, bits);
        qb.conv = quantize_rows(b.conv, e, bits);
        qb.out = quantize_rows(b.out_proj, e, bits);
        for (const DirW& d : b.dirs) {
            std::vector<double> xp(d.w_delta);
            xp.insert(xp.end(), d.w_b.begin(), d.w_b.end());
            xp.insert(xp.end(), d.w_c.begin(), d.w_c.end());
            qb.xp.push_back(quantize_rows(xp, e + 2 * n, bits));
        }
        q.blocks.push_back(std::move(qb));
    }
    return q;
}

template <class Ops>
struct Driver {
    const ModelW& m;
    const QModel* q;    // null in FP mode
    const Calib* cal;   // null in FP mode
    Mode mode;
    bool d1, d2;
    typename Ops::Prepared prep;  // per-model prepared GEMM weights (D2)

    Driver(const ModelW& model, const QModel* qm, const Calib* c, Mode md, bool D1, bool D2)
        : m(model), q(qm), cal(c), mode(md), d1(D1), d2(D2) {
        if (mode != MODE_FP) {
            require(q && cal, "quantized forward needs weights and calibration");
            require(cal->blocks == m.blocks.size() && cal->ndirs == m.orders.size() &&
                        cal->tokens == m.d.tokens() && cal->embed == m.d.embed,
                    "calibration does not match the model geometry");  // quant.cpp:508-510
            if (d2) require(cal->d2 && cal->lin.size() == cal->blocks * cal->nsites(),
                            "calibration lacks linear-input records (D2)");
            if (d2) prep = Ops::prepare(*q);
        }
    }

    // Weights the f64 paths multiply with: FP, or fake-quantized (quant.cpp:519).
    const double* wmat(const std::vector<double>& fp, const QRows* qr) const {
        return mode == MODE_FP ? fp.data() : qr->deq.data();
    }

    // Per-sample detector states, reset for every sample (quant.cpp:478-481).
    struct SampleState {
        std::vector<typename Ops::State> scan, lin;
    };
    SampleState fresh_state() const {
        SampleState s;
        s.scan.resize(m.blocks.size() * m.orders.size() * 3);
        s.lin.resize(m.blocks.size() * (m.orders.size() + 2));
        return s;
    }

    // QuantHook::apply, quant.cpp:467-491.
    bool policy(SampleState& ss, std::size_t b, std::size_t d, int kind, std::size_t t, double* x,
                std::size_t e, std::size_t n) const {
        if (mode == MODE_FP) return false;
        const TCal& tc = cal->at(b, d, kind);
        require(t < tc.s_in.size(), "quantized step beyond calibrated sequence length");
        if (mode == MODE_STATIC) {
            Ops::fake_quant(x, e, n, nullptr, tc.s_full[t], cal->spec.abits, cal->spec.obits);
            return false;
        }
        auto& st = ss.scan[(b * m.orders.size() + d) * 3 + kind];
        Ops::refresh(st, t, cal->spec.n_refresh);
        bool scanned = Ops::detect(st, x, e, n, tc.theta, tc.s_in[t], cal->spec.abits);
        Ops::fake_quant(x, e, n, &st, tc.s_in[t], cal->spec.abits, cal->spec.obits);
        return scanned;
    }

    // D2: one token plane through detect -> split_quantize -> hybrid GEMM.
    void quant_linear(SampleState& ss, std::size_t b, std::size_t site, std::size_t t, const double* x,
                      const typename Ops::Weight& w, double* out, LinTrace* tr, std::size_t R) const {
        std::size_t e = m.d.embed;
        const TCal& tc = cal->site(b, site);
        require(t < tc.s_in.size(), "quantized step beyond calibrated sequence length");
        std::vector<std::size_t> olist;
        double s;
        bool scanned = false;
        if (mode == MODE_STATIC) {
            s = tc.s_full[t];
        } else {
            auto& st = ss.lin[b * (m.orders.size() + 2) + site];
            Ops::refresh(st, t, cal->spec.n_refresh);
            scanned = Ops::detect(st, x, e, 1, tc.theta, tc.s_in[t], cal->spec.abits);
            olist = Ops::list(st, e);
            s = tc.s_in[t];
        }
        SplitOperands sp = Ops::split(x, e, 1, olist, s, cal->spec.abits, cal->spec.obits);
        GemmResult g = Ops::hybrid(w, sp, s);
        for (std::size_t r = 0; r < R; ++r) out[r] = g.output[r];
        if (tr) {
            std::memcpy(tr->codes.data() + t * e, sp.inlier_codes.data(), e);
            for (std::size_t j = 0; j < olist.size(); ++j) {
                std::size_t ch = olist[j];
                tr->omask[t * e + ch] = 1;
                tr->ocode[t * e + ch] = sp.outliers.codes[j];
                tr->oscale[t * e + ch] = sp.outliers.scales[j];
            }
            std::memcpy(tr->acc_in.data() + t * R, g.acc_inlier.data(), R * sizeof(std::int32_t));
            std::memcpy(tr->acc_out.data() + t * R, g.acc_outlier.data(), R * sizeof(std::int32_t));
            std::memcpy(tr->out.data() + t * R, g.output.data(), R * sizeof(double));
            tr->scanned[t] = scanned;
        }
    }

    static void init_lin(LinTrace& lt, std::size_t L, std::size_t E, std::size_t R) {
        lt.codes.assign(L * E, 0);
        lt.ocode.assign(L * E, 0);
        lt.omask.assign(L * E, 0);
        lt.oscale.assign(L * E, 0.0);
        lt.acc_in.assign(L * R, 0);
        lt.acc_out.assign(L * R, 0);
        lt.out.assign(L * R, 0.0);
        lt.scanned.assign(L, 0);
    }

    // s6_scan (ssm.cpp:124-186) with the QuantHook policy. With D2 the three
    // projections come precomputed from the quantized x_proj (proj: L x (E+2N)).
    void scan(SampleState& ss, std::size_t b, std::size_t d, const std::vector<double>& u,
              const double* proj, std::vector<double>& o, DirTrace* dt, Recorder* rec) const {
        const DirW& p = m.blocks[b].dirs[d];
        std::size_t L = m.d.tokens(), e = m.d.embed, n = m.d.state;
        const double* wdelta = nullptr;
        const double* wbv = nullptr;
        const double* wcv = nullptr;
        std::vector<double> wxp;
        if (!proj) {
            if (mode == MODE_FP) {
                wdelta = p.w_delta.data();
                wbv = p.w_b.data();
                wcv = p.w_c.data();
            } else {
                const QRows& qx = q->blocks[b].xp[d];
                wdelta = qx.deq.data();
                wbv = qx.deq.data() + e * e;
                wcv = qx.deq.data() + (e + n) * e;
            }
        }
        std::vector<double> h(e * n, 0.0), dproj(e), delta(e), bvec(n), cvec(n), a_bar(e * n), b_bar(e * n);
        o.assign(L * e, 0.0);
        for (std::size_t t = 0; t < L; ++t) {
            const double* ut = u.data() + t * e;
            if (proj) {
                const double* pr = proj + t * (e + 2 * n);
                for (std::size_t i = 0; i < e; ++i) delta[i] = Ops::softplus(pr[i] + p.b_delta[i]);
                for (std::size_t k = 0; k < n; ++k) bvec[k] = pr[e + k];
                for (std::size_t k = 0; k < n; ++k) cvec[k] = pr[e + n + k];
            } else {
                Ops::mm_nt(ut, wdelta, dproj.data(), 1, e, e);
                for (std::size_t i = 0; i < e; ++i) delta[i] = Ops::softplus(dproj[i] + p.b_delta[i]);
                Ops::mm_nt(ut, wbv, bvec.data(), 1, e, n);
                Ops::mm_nt(ut, wcv, cvec.data(), 1, e, n);
            }
            for (std::size_t i = 0; i < e; ++i)
                for (std::size_t k = 0; k < n; ++k) {
                    a_bar[i * n + k] = std::exp(delta[i] * p.a[i * n + k]);
                    b_bar[i * n + k] = delta[i] * bvec[k];
                }
            if (rec) {
                Recorder::note(rec->scan[(b * m.orders.size() + d) * 3 + ABAR], t, a_bar.data(), e, n);
                Recorder::note(rec->scan[(b * m.orders.size() + d) * 3 + BBAR], t, b_bar.data(), e, n);
            }
            bool sa = policy(ss, b, d, ABAR, t, a_bar.data(), e, n);
            bool sb = policy(ss, b, d, BBAR, t, b_bar.data(), e, n);
            if (dt) {
                dt->scanned[ABAR][t] = sa;
                dt->scanned[BBAR][t] = sb;
                record_mask(ss, b, d, ABAR, t, dt->mask[ABAR]);
                record_mask(ss, b, d, BBAR, t, dt->mask[BBAR]);
            }
            for (std::size_t i = 0; i < e; ++i)
                for (std::size_t k = 0; k < n; ++k)
                    h[i * n + k] = a_bar[i * n + k] * h[i * n + k] + b_bar[i * n + k] * ut[i];
            if (rec) Recorder::note(rec->scan[(b * m.orders.size() + d) * 3 + HST], t, h.data(), e, n);
            bool sh = policy(ss, b, d, HST, t, h.data(), e, n);
            if (dt) {
                dt->scanned[HST][t] = sh;
                record_mask(ss, b, d, HST, t, dt->mask[HST]);
            }
            for (std::size_t i = 0; i < e; ++i) {
                double s = 0.0;
                for (std::size_t k = 0; k < n; ++k) s += cvec[k] * h[i * n + k];
                o[t * e + i] = s;
            }
            if (dt) {
                std::memcpy(dt->delta.data() + t * e, delta.data(), e * sizeof(double));
                std::memcpy(dt->bvec.data() + t * n, bvec.data(), n * sizeof(double));
                std::memcpy(dt->cvec.data() + t * n, cvec.data(), n * sizeof(double));
            }
        }
        if (dt) {
            dt->u = u;
            dt->o = o;
        }
    }

    void record_mask(SampleState& ss, std::size_t b, std::size_t d, int kind, std::size_t t,
                     std::vector<std::uint8_t>& dst) const {
        if (mode != MODE_DYNAMIC) return;
        std::size_t e = m.d.embed;
        auto lst = Ops::list(ss.scan[(b * m.orders.size() + d) * 3 + kind], e);
        for (std::size_t ch : lst) dst[t * e + ch] = 1;
    }

    // One block over one sample's token matrix x (L x E), in place:
    // block_forward_raw, ssm.cpp:192-233, plus D1/D2.
    void block(SampleState& ss, std::size_t b, std::vector<double>& x, BlockTrace* bt, Recorder* rec) const {
        const BlockW& blk = m.blocks[b];
        std::size_t L = m.d.tokens(), e = m.d.embed, n = m.d.state, W = m.d.conv_width;
        std::size_t nd = m.orders.size();
        bool qlin = d2 && mode != MODE_FP;
        if (bt) {
            bt->x_in = x;
            bt->dirs.assign(nd, DirTrace{});
        }
        std::vector<double> xn(L * e);
        if (d1)
            for (std::size_t t = 0; t < L; ++t) rmsnorm_row(x.data() + t * e, xn.data() + t * e, e);
        else
            xn = x;
        if (rec && d2)
            for (std::size_t t = 0; t < L; ++t) Recorder::note(rec->lin[b * (nd + 2) + 0], t, xn.data() + t * e, e, 1);

        std::vector<double> gate(L * e), u0(L * e), u(L * e, 0.0);
        if (qlin) {
            std::vector<double> out(2 * e);
            LinTrace* lt = bt ? &bt->lin[0] : nullptr;
            if (lt) init_lin(*lt, L, e, 2 * e);
            for (std::size_t t = 0; t < L; ++t) {
                quant_linear(ss, b, 0, t, xn.data() + t * e, prep.blocks[b].in, out.data(), lt, 2 * e);
                for (std::size_t i = 0; i < e; ++i) {
                    u0[t * e + i] = out[i];
                    if (bt) bt->gpre.push_back(out[e + i]);
                    gate[t * e + i] = Ops::silu(out[e + i]);
                }
            }
        } else {
            const double* wg = mode == MODE_FP ? blk.w_gate.data() : q->blocks[b].in.deq.data() + e * e;
            const double* wi = mode == MODE_FP ? blk.w_in.data() : q->blocks[b].in.deq.data();
            Ops::mm_nt(xn.data(), wg, gate.data(), L, e, e);
            if (bt) bt->gpre = gate;
            for (double& v : gate) v = Ops::silu(v);
            Ops::mm_nt(xn.data(), wi, u0.data(), L, e, e);
        }
        // Depthwise causal conv, ssm.cpp:200-212.
        const double* taps = wmat(blk.conv, q ? &q->blocks[b].conv : nullptr);
        for (std::size_t t = 0; t < L; ++t)
            for (std::size_t c = 0; c < e; ++c) {
                double s = 0.0;
                for (std::size_t k = 0; k < W; ++k) {
                    std::int64_t src = static_cast<std::int64_t>(t) - static_cast<std::int64_t>(W - 1 - k);
                    if (src < 0) continue;
                    s += taps[c * W + k] * u0[static_cast<std::size_t>(src) * e + c];
                }
                u[t * e + c] = s;
            }
        if (bt) {
            bt->xn = xn;
            bt->u0 = u0;
            bt->gate = gate;
            bt->u = u;
        }
        // Directions: permute -> scan -> unpermute and merge by sum, ssm.cpp:214-229.
        std::vector<double> merged(L * e, 0.0);
        for (std::size_t d = 0; d < nd; ++d) {
            auto perm = scan_permutation(m.orders[d], m.d.grid());
            std::vector<double> up(L * e);
            for (std::size_t t = 0; t < L; ++t)
                std::memcpy(up.data() + t * e, u.data() + perm[t] * e, e * sizeof(double));
            DirTrace* dt = bt ? &bt->dirs[d] : nullptr;
            if (dt) {
                dt->delta.assign(L * e, 0.0);
                dt->bvec.assign(L * n, 0.0);
                dt->cvec.assign(L * n, 0.0);
                for (int k = 0; k < 3; ++k) {
                    dt->mask[k].assign(L * e, 0);
                    dt->scanned[k].assign(L, 0);
                }
            }
            if (rec && d2)
                for (std::size_t t = 0; t < L; ++t)
                    Recorder::note(rec->lin[b * (nd + 2) + 1 + d], t, up.data() + t * e, e, 1);
            std::vector<double> proj;
            if (qlin) {
                std::size_t R = e + 2 * n;
                proj.resize(L * R);
                LinTrace* lt = bt ? &bt->lin[1 + d] : nullptr;
                if (lt) init_lin(*lt, L, e, R);
                for (std::size_t t = 0; t < L; ++t)
                    quant_linear(ss, b, 1 + d, t, up.data() + t * e, prep.blocks[b].xp[d], proj.data() + t * R, lt, R);
            }
            std::vector<double> o;
            scan(ss, b, d, up, qlin ? proj.data() : nullptr, o, dt, rec);
            for (std::size_t t = 0; t < L; ++t) {
                const double* src = o.data() + t * e;
                double* dst = merged.data() + perm[t] * e;
                for (std::size_t i = 0; i < e; ++i) dst[i] += src[i];
            }
        }
        std::vector<double> y(L * e);
        for (std::size_t i = 0; i < L * e; ++i) y[i] = merged[i] * gate[i];
        if (rec && d2)
            for (std::size_t t = 0; t < L; ++t) Recorder::note(rec->lin[b * (nd + 2) + nd + 1], t, y.data() + t * e, e, 1);
        std::vector<double> out(L * e);
        if (qlin) {
            LinTrace* lt = bt ? &bt->lin[nd + 1] : nullptr;
            if (lt) init_lin(*lt, L, e, e);
            for (std::size_t t = 0; t < L; ++t)
                quant_linear(ss, b, nd + 1, t, y.data() + t * e, prep.blocks[b].out, out.data() + t * e, lt, e);
        } else {
            Ops::mm_nt(y.data(), wmat(blk.out_proj, q ? &q->blocks[b].out : nullptr), out.data(), L, e, e);
        }
        if (d1)
            for (std::size_t i = 0; i < L * e; ++i) x[i] = x[i] + out[i];
        else
            x = out;
        if (bt) {
            bt->merged = merged;
            bt->y = y;
            bt->x_out = x;
        }
    }

    // vmm_forward_raw for one sample, ssm.cpp:250-275.
    void sample(const double* img, double* logits, std::size_t trace_block, BlockTrace* bt, Recorder* rec,
                std::vector<double>* x_embed = nullptr) const {
        const Dims& d = m.d;
        std::size_t L = d.tokens(), e = d.embed, pv = d.patch_vals();
        auto gather = patch_gather_indices(d);
        std::vector<double> patches(L * pv), x(L * e), pooled(e, 0.0), lg(d.classes);
        for (std::size_t i = 0; i < L * pv; ++i) patches[i] = img[gather[i]];
        Ops::mm_nt(patches.data(), wmat(m.patch_w, q ? &q->patch : nullptr), x.data(), L, pv, e);
        for (std::size_t t = 0; t < L; ++t)
            for (std::size_t i = 0; i < e; ++i) x[t * e + i] += m.patch_b[i];
        if (x_embed) *x_embed = x;
        SampleState ss = fresh_state();
        for (std::size_t b = 0; b < m.blocks.size(); ++b)
            block(ss, b, x, b == trace_block ? bt : nullptr, rec);
        for (std::size_t t = 0; t < L; ++t)
            for (std::size_t i = 0; i < e; ++i) pooled[i] += x[t * e + i];
        double inv_m = 1.0 / static_cast<double>(L);
        for (double& v : pooled) v *= inv_m;
        Ops::mm_nt(pooled.data(), wmat(m.head_w, q ? &q->head : nullptr), lg.data(), 1, e, d.classes);
        for (std::size_t c = 0; c < d.classes; ++c) logits[c] = lg[c] + m.head_b[c];
    }

    // Batch forward: samples are independent (per-sample state, quant.cpp:477-481),
    // so a static partition over threads is exact.
    void batch(const double* images, std::size_t B, double* logits, int threads, Recorder* rec) const {
        std::size_t pix = m.d.image * m.d.image * m.d.channels;
        std::size_t T = std::max<std::size_t>(1, std::min<std::size_t>(threads < 1 ? 1 : threads, B));
        std::vector<std::unique_ptr<Recorder>> recs(T);
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(T);
        for (std::size_t w = 0; w < T; ++w) {
            if (rec) recs[w] = std::make_unique<Recorder>(rec->tokens, rec->embed, rec->scan.size(), rec->lin.size());
            pool.emplace_back([&, w] {
                try {
                    for (std::size_t s = w; s < B; s += T)
                        sample(images + s * pix, logits + s * m.d.classes, SIZE_MAX, nullptr, rec ? recs[w].get() : nullptr);
                } catch (...) {
                    errs[w] = std::current_exception();
                }
            });
        }
        for (auto& t : pool) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        if (rec)
            for (auto& r : recs) rec->merge(*r);
    }
};

// calibrate, quant.cpp:129-177 (+ D2 sites): FP forward with the recorder.
template <class Ops>
Calib calibrate(const ModelW& m, const double* images, std::size_t B, const Spec& spec, bool d1, bool d2,
                int threads) {
    spec.validate();
    std::size_t L = m.d.tokens(), E = m.d.embed, nd = m.orders.size(), nb = m.blocks.size();
    Recorder rec(L, E, nb * nd * 3, d2 ? nb * (nd + 2) : 0);
    Driver<Ops> drv(m, nullptr, nullptr, MODE_FP, d1, d2);
    std::vector<double> logits(B * m.d.classes);
    drv.batch(images, B, logits.data(), threads, &rec);
    Calib c;
    c.spec = spec;
    c.tokens = L;
    c.embed = E;
    c.state = m.d.state;
    c.blocks = nb;
    c.ndirs = nd;
    c.d1 = d1;
    c.d2 = d2;
    for (auto& pk : rec.scan) c.scan.push_back(reduce_calib(pk, L, E, spec.rho, spec.abits));
    for (auto& pk : rec.lin) c.lin.push_back(reduce_calib(pk, L, E, spec.rho, spec.abits));
    return c;
}

}  // namespace oro
