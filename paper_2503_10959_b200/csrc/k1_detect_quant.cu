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
// Output operand (QAct): codes [M][E] (0 at outliers), per-row mask words
// [M][J] (bit ch%32 of word ch/32 = channel in O(t)), dense outlier codes and
// scales [M][E] written at outlier positions only, |O(t)| per row and the
// row's inlier scale. The hybrid epilogue walks the mask words in ascending
// channel order, the order the reference adds outlier terms in
// (gemm.cpp:208-216).
//
// Two kernels:
//  * k1_channel (fast path): one thread owns four channels of one (sample,
//    refresh window) and walks the window's tokens. Exact whenever
//    C(t) = fl(nextafter(theta,+inf)/q_a) > S^I(t) holds (host-checked per
//    site and step): then O(t) = O_r(t) U {ch: |x| > theta}
//    and channels never interact. Rows are read as 16-byte vectors, codes
//    stored as char4; D1's RMSNorm factor comes from k1_rownorm.
//  * k1_literal: one warp owns one (sample, window) with lane l holding
//    channels l, l+32, ...; the cross-channel maximum of detect_outliers is a
//    warp reduction, so the reference is followed verbatim (also provides
//    DetectResult::scanned).
#include "common.cuh"
#include "kernels.h"

namespace ob {

// D1 RMSNorm factor per token row: 1/sqrt(mean(x^2) + 1e-6) with the sum taken
// as 32 lane-strided partials (channel k -> partial k%32, k ascending) combined
// by an xor butterfly (oracle/driver.hpp rmsnorm_row).
__global__ void __launch_bounds__(256) k1_rownorm(const double* __restrict__ x, double* __restrict__ rs, long rows,
                                                  int E) {
    const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const double* xr = x + r * E;
    double ps = 0.0;
    int k = lane;
    for (; k + 7 * 32 < E; k += 8 * 32) {  // 8 loads in flight, summed in channel order
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldg(xr + k + 32 * j);
#pragma unroll
        for (int j = 0; j < 8; ++j) ps = dadd(ps, dmul(v[j], v[j]));
    }
    for (; k < E; k += 32) {
        const double v = __ldg(xr + k);
        ps = dadd(ps, dmul(v, v));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ps = dadd(ps, __shfl_xor_sync(0xffffffffu, ps, o));
    if (lane == 0) {
        const double ms = __ddiv_rn(ps, static_cast<double>(E));
        rs[r] = __ddiv_rn(1.0, __dsqrt_rn(dadd(ms, 1e-6)));
    }
}

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

// Layer input of two channels at one token (16-byte loads).
template <int SRC>
__device__ __forceinline__ double2 k1_load2(const K1Params& p, size_t src, size_t crow_global) {
    if (SRC == K1_SRC_MERGE) {
        // merged = (0 + o_0) + o_1 (ssm.cpp:214-229), y = merged * gate (ssm.cpp:231)
        const double2 a = ldg2(p.x + src);
        const double2 g = ldg2(p.gate + src);
        double m0 = dadd(0.0, a.x), m1 = dadd(0.0, a.y);
        if (p.x2) {
            const double2 b = ldg2(p.x2 + src);
            m0 = dadd(m0, b.x);
            m1 = dadd(m1, b.y);
        }
        return make_double2(dmul(m0, silu_d(g.x)), dmul(m1, silu_d(g.y)));  // gate = silu(x W_g^T)
    }
    double2 v = ldg2(p.x + src);
    if (SRC == K1_SRC_RMSNORM) {
        const double r = __ldg(p.rs + crow_global);
        v.x = dmul(v.x, r);
        v.y = dmul(v.y, r);
    }
    return v;
}

// Merge source, certified form. v = m * silu(g) with m = (0 + o_0) + o_1 exact
// in f64; v is evaluated in f32 with a relative error bound, and the detector
// decision and inlier code are taken from it only when the bound keeps them
// away from theta and from half-integers; otherwise (and for outlier channels)
// the exact f64 value is used. Bound: g and m rounded to f32 (2 x 2^-24),
// the ex2 argument (3|g| 2^-24 relative in e), ex2.approx (2^-22), the
// sigmoid's add and quotient (2 x 2^-24, doubled for g < 0 where e/(1+e)
// carries e's error in full), two products: |vf/v - 1| <= (6|g| + 15) 2^-24;
// the code adds 1/s rounded to f32 and one product. Below g = -80 ex2 flushes,
// so those elements always take the exact path.
struct MergeApprox {
    float v, eps;
};
// exact merged value y = merged * silu(gate) (ssm.cpp:231): the rare path, kept out of line
__device__ __noinline__ double merge_exact(double m, double g) { return dmul(m, silu_d(g)); }
__device__ __forceinline__ MergeApprox merge_approx(double m, double g) {
    const float gf = __double2float_rn(g), mf = __double2float_rn(m);
    const float ag = fabsf(gf);
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-ag * 1.44269504f));
    const float den = 1.0f + e;
    const float sig = (gf >= 0.0f ? 1.0f : e) / den;
    MergeApprox r;
    r.v = (mf * gf) * sig;
    if (m == 0.0 || g == 0.0) {  // v = +-0 exactly: code 0, never an outlier (frequent: all-zero h codes)
        r.v = 0.0f;
        r.eps = 0.0f;
        return r;
    }
    // f32 subnormals (relative error unbounded), the ex2 flush and overflow take the exact path
    const bool ok = gf >= -80.0f && ag >= 1e-30f && fabsf(mf) >= 1e-30f && fabsf(r.v) < 1e30f;
    r.eps = ok ? fmaf(ag, 6.0f, 24.0f) * 5.9604645e-8f : 1.0f;
    return r;
}

// One thread owns four channels of one (sample, refresh window) and walks the
// window's tokens; a warp covers 128 channels = 4 mask words (8 lanes x 4 bits).
template <int SRC>
__global__ void __launch_bounds__(256) k1_channel(const K1Params p) {
    const int E = p.E, T = p.T, J = E >> 5;
    const int ch = (blockIdx.x * blockDim.x + threadIdx.x) * 4;  // channels ch .. ch+3
    const int lane = threadIdx.x & 31;
    const int win = p.window, nwin = (T + win - 1) / win;
    const int s = blockIdx.y / nwin;
    const int t0 = (blockIdx.y % nwin) * win, t1 = min(T, t0 + win);
    const bool active = ch < E;  // E is a multiple of 32
    const bool dyn = p.mode == MODE_DYNAMIC;
    const double qa = qmax_for(p.abits), qo = qmax_for(p.obits);
    const int qai = static_cast<int>(qa);
    const double theta = p.cal.theta;
    const float thetaf = __double2float_rn(theta);
    const double* __restrict__ s_tab = dyn ? p.cal.s_in : p.cal.s_full;
    const double* __restrict__ i_tab = dyn ? p.inv_in : p.inv_full;
    // maybe_refresh points inside the window (t0 is 0 or a refresh point, where the
    // state starts clear anyway)
    int next_ref = (dyn && p.n_refresh > 0) ? t0 + p.n_refresh : 0x7fffffff;
    unsigned in = 0;  // bit k: channel ch+k is in O
    for (int t = t0; t < t1; ++t) {
        const int crow = p.order <= 0 ? t : (p.order == 1 ? T - 1 - t : scan_perm(p.order, t, p.grid));
        const size_t cg = static_cast<size_t>(s) * T + crow;
        const size_t row = static_cast<size_t>(s) * T + t;
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        double mg[4], gg[4];  // merge source: merged scan output and gate pre-activation
        MergeApprox ap[4];
        if (active) {
            if (SRC == K1_SRC_MERGE) {
                const size_t src = cg * E + ch;
                const double2 a0 = ldg2(p.x + src), a1 = ldg2(p.x + src + 2);
                const double2 g0 = ldg2(p.gate + src), g1 = ldg2(p.gate + src + 2);
                mg[0] = dadd(0.0, a0.x);  // (0 + o_0) + o_1, ssm.cpp:214-229
                mg[1] = dadd(0.0, a0.y);
                mg[2] = dadd(0.0, a1.x);
                mg[3] = dadd(0.0, a1.y);
                if (p.x2) {
                    const double2 b0 = ldg2(p.x2 + src), b1 = ldg2(p.x2 + src + 2);
                    mg[0] = dadd(mg[0], b0.x);
                    mg[1] = dadd(mg[1], b0.y);
                    mg[2] = dadd(mg[2], b1.x);
                    mg[3] = dadd(mg[3], b1.y);
                }
                gg[0] = g0.x;
                gg[1] = g0.y;
                gg[2] = g1.x;
                gg[3] = g1.y;
#pragma unroll
                for (int k = 0; k < 4; ++k) ap[k] = merge_approx(mg[k], gg[k]);
            } else {
                const double2 lo = k1_load2<SRC>(p, cg * E + ch, cg), hi = k1_load2<SRC>(p, cg * E + ch + 2, cg);
                v[0] = lo.x;
                v[1] = lo.y;
                v[2] = hi.x;
                v[3] = hi.y;
            }
        }
        unsigned have = 0;  // merge: bit k = v[k] holds the exact value
        if (dyn) {
            if (t == next_ref) {  // maybe_refresh
                in = 0;
                next_ref += p.n_refresh;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // detect_outliers, channel-local form
                if (SRC == K1_SRC_MERGE) {
                    if (!active || ((in >> k) & 1u)) continue;
                    const float av = fabsf(ap[k].v);
                    if (av * (1.0f - ap[k].eps) > thetaf * 1.0000003f) {
                        in |= 1u << k;
                    } else if (av * (1.0f + ap[k].eps) >= thetaf * 0.9999997f) {
                        v[k] = merge_exact(mg[k], gg[k]);
                        have |= 1u << k;
                        if (fabs(v[k]) > theta) in |= 1u << k;
                    }
                } else {
                    if (fabs(v[k]) > theta) in |= 1u << k;
                }
            }
        }
        const double S = s_tab[t];
        const double inv = i_tab ? i_tab[t] : __ddiv_rn(1.0, S);
        if (active) {
            int c[4];
            const float invf = __double2float_rn(inv), capf = static_cast<float>(qa) + 1.0f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                c[k] = 0;
                if ((in >> k) & 1u) {
                    if (SRC == K1_SRC_MERGE && !((have >> k) & 1u)) v[k] = merge_exact(mg[k], gg[k]);
                    const double os = scale_from_peak(fabs(v[k]), qo);  // scale_for over the 1-value row
                    p.ocode[row * E + ch + k] = static_cast<int8_t>(static_cast<int>(quant_code_div(v[k], os, qo)));
                    p.oscale[row * E + ch + k] = os;
                } else if (SRC == K1_SRC_MERGE) {
                    // certified f32 quotient: |dq| <= (|q| + 1) (eps + 3 2^-24)
                    const float q = fminf(fmaxf(ap[k].v * invf, -capf), capf);
                    const float r = rintf(q);
                    if (!((have >> k) & 1u) &&
                        fabsf(q - r) < 0.5f - fmaf(fabsf(q) + 1.0f, ap[k].eps + 1.8e-7f, 1e-6f)) {
                        c[k] = min(max(static_cast<int>(r), -qai), qai);
                    } else {
                        if (!((have >> k) & 1u)) v[k] = merge_exact(mg[k], gg[k]);
                        c[k] = quant_code_int(v[k], S, inv, qa, qai);
                    }
                } else {
                    c[k] = quant_code_int(v[k], S, inv, qa, qai);
                }
            }
            *reinterpret_cast<char4*>(p.codes + row * E + ch) =
                make_char4(static_cast<signed char>(c[0]), static_cast<signed char>(c[1]),
                           static_cast<signed char>(c[2]), static_cast<signed char>(c[3]));
        }
        // mask word of channels 32w..32w+31 from 8 lanes x 4 bits (all zero in the common case)
        unsigned bits = active ? in << ((lane & 7) * 4) : 0u;
        if (__any_sync(0xffffffffu, bits != 0u)) {
#pragma unroll
            for (int o = 4; o >= 1; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
        }
        if (active && (lane & 7) == 0) {
            p.omask[row * J + (ch >> 5)] = bits;
            if (bits) atomicAdd(p.ocnt + row, __popc(bits));
        }
        if (ch == 0) p.s_row[row] = S;
    }
}

template <int JMAX, int SRC>
__global__ void __launch_bounds__(256) k1_literal(const K1Params p) {
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
                    double m = dadd(0.0, p.x[src + ch]);
                    if (p.x2) m = dadd(m, p.x2[src + ch]);
                    x = dmul(m, silu_d(p.gate[src + ch]));
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
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < JMAX; ++j) {
            const int ch = j * 32 + lane;
            const bool valid = j < J && ch < E;
            const bool isout = valid && ((inmask >> j) & 1u);
            if (valid) {
                double c = 0.0;
                if (isout) {
                    const double os = scale_from_peak(fabs(v[j]), qo);
                    p.ocode[row * E + ch] = static_cast<int8_t>(static_cast<int>(quant_code_div(v[j], os, qo)));
                    p.oscale[row * E + ch] = os;
                } else {
                    c = quant_code_inv(v[j], S, inv, qa);
                }
                p.codes[row * E + ch] = static_cast<int8_t>(static_cast<int>(c));
            }
            if (j < J) {
                const unsigned mb = __ballot_sync(0xffffffffu, isout);
                cnt += __popc(mb);
                if (lane == 0) p.omask[row * J + j] = mb;
            }
        }
        if (lane == 0) {
            p.ocnt[row] = cnt;
            p.s_row[row] = S;
            if (p.scanned) p.scanned[row] = trig ? 1 : 0;
        }
    }
}

template <int SRC>
static cudaError_t launch_literal(const K1Params& p, cudaStream_t st) {
    const int J = (p.E + 31) / 32;
    const int nwin = (p.T + p.window - 1) / p.window;
    const long warps = static_cast<long>(p.S) * nwin;
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>((warps * 32 + threads - 1) / threads);
    if (J <= 8) k1_literal<8, SRC><<<blocks, threads, 0, st>>>(p);
    else if (J <= 16) k1_literal<16, SRC><<<blocks, threads, 0, st>>>(p);
    else if (J <= 24) k1_literal<24, SRC><<<blocks, threads, 0, st>>>(p);
    else if (J <= 32) k1_literal<32, SRC><<<blocks, threads, 0, st>>>(p);
    else return cudaErrorInvalidValue;
    ++kernel_launch_counter();
    return cudaGetLastError();
}

template <int SRC>
static cudaError_t launch_channel(const K1Params& p, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(p.ocnt, 0, static_cast<size_t>(p.S) * p.T * sizeof(int), st);
    if (e != cudaSuccess) return e;
    if (SRC == K1_SRC_RMSNORM) {
        const long rows = static_cast<long>(p.S) * p.T;
        k1_rownorm<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(p.x, p.rs, rows, p.E);
        ++kernel_launch_counter();
    }
    const int nwin = (p.T + p.window - 1) / p.window;
    const int quads = p.E / 4, threads = quads >= 256 ? 256 : ((quads + 31) / 32) * 32;
    dim3 grid((quads + threads - 1) / threads, p.S * nwin);
    k1_channel<SRC><<<grid, threads, 0, st>>>(p);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

cudaError_t launch_k1(const K1Params& p, cudaStream_t st) {
    if (p.E < 1 || p.E > 1024 || p.T < 1 || p.S < 1 || p.window < 1) return cudaErrorInvalidValue;
    // the channel-parallel kernel needs: a quantizing mode, no DetectResult
    // output, the channel-local detector exact (no literal steps), E % 32 == 0
    // and (RMSNORM) a row-factor buffer
    const bool fast = p.mode != MODE_FP && !p.scanned && !p.force_literal && (p.E % 32) == 0 &&
                      (p.src != K1_SRC_RMSNORM || p.rs != nullptr);
    switch (p.src) {
        case K1_SRC_PLAIN: return fast ? launch_channel<K1_SRC_PLAIN>(p, st) : launch_literal<K1_SRC_PLAIN>(p, st);
        case K1_SRC_RMSNORM:
            return fast ? launch_channel<K1_SRC_RMSNORM>(p, st) : launch_literal<K1_SRC_RMSNORM>(p, st);
        case K1_SRC_MERGE: return fast ? launch_channel<K1_SRC_MERGE>(p, st) : launch_literal<K1_SRC_MERGE>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ob
