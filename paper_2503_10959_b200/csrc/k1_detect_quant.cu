// K1 — per-time-step dynamic outlier detector fused with activation
// quantization, for the inputs of the quant-linear layers (in_proj, x_proj per
// direction, out_proj).
//
// Reference semantics restated (per (sample, token) plane of E channels x 1
// column, DESIGN.md §2 D2):
//   maybe_refresh      quant.cpp:303-311   clear O before detection at t
//   detect_outliers    quant.cpp:313-335   s_dyn = max_{ch not in O}|x|/q_a;
//                                          if s_dyn > S^I(t): O |= {ch: |x| > theta}
//   split_quantize     gemm.cpp:106-135    inliers -> code(x, S^I(t), a_bits),
//                                          outliers -> own scale |x|/q_o, code at o_bits
// Layout/work split: one warp owns one (sample, refresh window); lane l owns
// channels l, l+32, ... (so every cross-channel quantity of the reference —
// the detector's max, D1's RMSNorm sum — is a warp shuffle reduction), and the
// warp walks the window's tokens in step order carrying O as a per-lane bit
// mask. Rows are read with 256 B coalesced loads; the outlier list of every
// row is compacted in ascending channel order with ballots, which is the order
// the hybrid epilogue adds outlier terms in (gemm.cpp:208-216).
#include "common.cuh"
#include "kernels.h"

namespace ob {

template <int JMAX, int SRC>
__global__ void __launch_bounds__(256) k1_detect_quant(const K1Params p) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int win = p.window;
    const int nwin = (p.T + win - 1) / win;
    if (gw >= p.S * nwin) return;
    const int s = gw / nwin;
    const int t0 = (gw % nwin) * win;
    const int t1 = min(p.T, t0 + win);
    const int E = p.E;
    const int J = (E + 31) >> 5;
    const double qa = qmax_for(p.abits), qo = qmax_for(p.obits);
    unsigned inmask = 0;  // bit j: channel j*32+lane is in O

    for (int t = t0; t < t1; ++t) {
        const int crow = p.order < 0 ? t : scan_perm(p.order, t, p.grid);
        const size_t src = (static_cast<size_t>(s) * p.T + crow) * E;
        const size_t row = static_cast<size_t>(s) * p.T + t;
        double v[JMAX];
#pragma unroll
        for (int j = 0; j < JMAX; ++j) {
            const int ch = j * 32 + lane;
            double x = 0.0;
            if (j < J && ch < E) {
                if (SRC == K1_SRC_MERGE) {
                    // merged = (0 + o_0) + o_1 (ssm.cpp:214-229), y = merged * gate (ssm.cpp:231)
                    double m = dadd(0.0, p.x[src + ch]);
                    if (p.x2) m = dadd(m, p.x2[src + ch]);
                    x = dmul(m, p.gate[src + ch]);
                } else {
                    x = p.x[src + ch];
                }
            }
            v[j] = x;
        }
        if (SRC == K1_SRC_RMSNORM) {  // D1: lane-strided partials + xor butterfly
            double ps = 0.0;
#pragma unroll
            for (int j = 0; j < JMAX; ++j)
                if (j < J && j * 32 + lane < E) ps = dadd(ps, dmul(v[j], v[j]));
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) ps = dadd(ps, __shfl_xor_sync(0xffffffffu, ps, o));
            const double ms = __ddiv_rn(ps, static_cast<double>(E));
            const double r = __ddiv_rn(1.0, __dsqrt_rn(dadd(ms, 1e-6)));
#pragma unroll
            for (int j = 0; j < JMAX; ++j) v[j] = dmul(v[j], r);
        }
        if (p.mode == MODE_FP) {  // materialize the layer input and record calibration peaks
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                const int ch = j * 32 + lane;
                if (j < J && ch < E) {
                    if (p.xout) p.xout[row * E + ch] = v[j];
                    if (p.peaks)
                        atomicMax(p.peaks + static_cast<size_t>(t) * E + ch,
                                  static_cast<unsigned long long>(__double_as_longlong(fabs(v[j]))));
                }
            }
            continue;
        }
        double S;
        bool trig = false;
        if (p.mode == MODE_DYNAMIC) {
            if (refresh_at(t, p.n_refresh)) inmask = 0;
            double mx = 0.0;
#pragma unroll
            for (int j = 0; j < JMAX; ++j)
                if (!((inmask >> j) & 1u)) mx = fmax(mx, fabs(v[j]));
            mx = warp_max(mx);
            S = p.cal.s_in[t];
            trig = !(__ddiv_rn(mx, qa) <= S);
            if (trig) {
#pragma unroll
                for (int j = 0; j < JMAX; ++j) {
                    const int ch = j * 32 + lane;
                    if (j < J && ch < E && fabs(v[j]) > p.cal.theta) inmask |= 1u << j;
                }
            }
        } else {
            S = p.cal.s_full[t];
        }
        const double inv = __ddiv_rn(1.0, S);
        int base = 0;
        int8_t* crow_codes = p.codes + row * E;
#pragma unroll
        for (int j = 0; j < JMAX; ++j) {
            const int ch = j * 32 + lane;
            const bool valid = j < J && ch < E;
            const bool isout = valid && ((inmask >> j) & 1u);
            if (valid) {
                double c = 0.0;
                if (!isout) c = quant_code_inv(v[j], S, inv, qa);
                crow_codes[ch] = static_cast<int8_t>(static_cast<int>(c));
            }
            const unsigned bal = __ballot_sync(0xffffffffu, isout);
            if (bal) {
                if (isout) {
                    const int pos = base + __popc(bal & ((1u << lane) - 1u));
                    const double ap = fabs(v[j]);
                    const double os = scale_from_peak(ap, qo);  // scale_for over the 1-value row
                    const double oc = quant_code_div(v[j], os, qo);
                    const size_t o = row * p.cap + pos;
                    p.och[o] = static_cast<uint16_t>(ch);
                    p.ocode[o] = static_cast<int8_t>(static_cast<int>(oc));
                    p.oscale[o] = os;
                }
                base += __popc(bal);
            }
            if (p.omask && j < J) {
                const unsigned mb = __ballot_sync(0xffffffffu, isout);
                if (lane == 0) p.omask[row * J + j] = mb;
            }
        }
        if (lane == 0) {
            p.ocnt[row] = base;
            p.s_row[row] = S;
            if (p.scanned) p.scanned[row] = trig ? 1 : 0;
        }
    }
}

template <int SRC>
static cudaError_t launch_src(const K1Params& p, cudaStream_t st) {
    const int J = (p.E + 31) / 32;
    const int nwin = (p.T + p.window - 1) / p.window;
    const long warps = static_cast<long>(p.S) * nwin;
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>((warps * 32 + threads - 1) / threads);
    if (J <= 8) k1_detect_quant<8, SRC><<<blocks, threads, 0, st>>>(p);
    else if (J <= 16) k1_detect_quant<16, SRC><<<blocks, threads, 0, st>>>(p);
    else if (J <= 24) k1_detect_quant<24, SRC><<<blocks, threads, 0, st>>>(p);
    else if (J <= 32) k1_detect_quant<32, SRC><<<blocks, threads, 0, st>>>(p);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

cudaError_t launch_k1(const K1Params& p, cudaStream_t st) {
    if (p.E < 1 || p.E > 1024 || p.T < 1 || p.S < 1 || p.window < 1) return cudaErrorInvalidValue;
    switch (p.src) {
        case K1_SRC_PLAIN: return launch_src<K1_SRC_PLAIN>(p, st);
        case K1_SRC_RMSNORM: return launch_src<K1_SRC_RMSNORM>(p, st);
        case K1_SRC_MERGE: return launch_src<K1_SRC_MERGE>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ob
