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
// Three kernels:
//  * k1_staged (fast path, plain / RMSNorm sources): a CTA owns one (sample,
//    refresh window) and all E channels; the window's rows arrive in shared
//    memory by bulk copies (two-stage ring, any scan order), D1's row factor is
//    taken from the staged rows, and one thread walks four channels. Both scan
//    directions' x_proj inputs can share one launch (CTAs interleaved so
//    mirrored windows read the same rows from L2).
//  * k1_channel (fast path, merge source): one thread owns four channels of
//    one (sample, refresh window) and walks the window's tokens. Both fast
//    kernels are exact whenever
//    C(t) = fl(nextafter(theta,+inf)/q_a) > S^I(t) holds (host-checked per
//    site and step): then O(t) = O_r(t) U {ch: |x| > theta}
//    and channels never interact. Rows are read as 16-byte vectors, codes
//    stored as char4; D1's RMSNorm factor is taken from the staged rows
//    (k1_staged), so x is read once.
//  * k1_literal: one warp owns one (sample, window) with lane l holding
//    channels l, l+32, ...; the cross-channel maximum of detect_outliers is a
//    warp reduction, so the reference is followed verbatim (also provides
//    DetectResult::scanned).
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "merge_f32.cuh"
#include "sm100_ptx.cuh"

namespace ob {

// channels per thread of the merge K1 (k1_channel): 4 (Vim-B batch 256: 217 us per launch;
// 2 channels per thread, 60 registers and a third more warps, measured 267 us)
#ifndef K1_MERGE_CPT
#define K1_MERGE_CPT 4
#endif

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

// four consecutive codes in [-7, 7] as two pack_int4 bytes (gemm.cpp:60-73: low nibble
// = even column), one 16-bit store
__device__ __forceinline__ uint16_t pack4(int c0, int c1, int c2, int c3) {
    return static_cast<uint16_t>((c0 & 0xF) | ((c1 & 0xF) << 4) | ((c2 & 0xF) << 8) | ((c3 & 0xF) << 12));
}


// |a|, |b|, |c| or |d| > th as one predicate chain (setp.gt.or)
__device__ __forceinline__ bool any_abs_gt4(double a, double b, double c, double d, double th) {
    unsigned r;
    asm("{\n\t.reg .pred p;\n\t.reg .f64 x;\n\t"
        "abs.f64 x, %1;\n\tsetp.gt.f64 p, x, %5;\n\t"
        "abs.f64 x, %2;\n\tsetp.gt.or.f64 p, x, %5, p;\n\t"
        "abs.f64 x, %3;\n\tsetp.gt.or.f64 p, x, %5, p;\n\t"
        "abs.f64 x, %4;\n\tsetp.gt.or.f64 p, x, %5, p;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r) : "d"(a), "d"(b), "d"(c), "d"(d), "d"(th));
    return r != 0u;
}

// exact merged value y = merged * silu(gate) (ssm.cpp:231): the rare path, kept out of line
__device__ __noinline__ double merge_exact(double m, double g) { return dmul(m, silu_d(g)); }

// One thread owns four channels of one (sample, refresh window) and walks the
// window's tokens; a warp covers 128 channels = 4 mask words (8 lanes x 4 bits).
template <int SRC, int CPT>
__global__ void __launch_bounds__(256) k1_channel(const K1Params p) {
    static_assert(SRC == K1_SRC_MERGE, "plain and RMSNorm sources run on k1_staged");
    static_assert(CPT == 2 || CPT == 4, "two or four channels per thread");
    constexpr int kLanesPerWord = 32 / CPT;
    const int E = p.E, T = p.T, J = E >> 5;
    const int ch = (blockIdx.x * blockDim.x + threadIdx.x) * CPT;  // channels ch .. ch+CPT-1
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
        const int crow = row_at(p.order, t, T, p.grid);
        const size_t cg = static_cast<size_t>(s) * T + crow;
        const size_t row = static_cast<size_t>(s) * T + t;
        double v[CPT], mg[CPT], gg[CPT];  // merge source: merged scan output and gate pre-activation
        MergeApprox ap[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) v[k] = 0.0;
        if (active) {
            const size_t src = cg * E + ch;
#pragma unroll
            for (int h = 0; h < CPT / 2; ++h) {
                const double2 a = ldg2(p.x + src + 2 * h), g = ldg2(p.gate + src + 2 * h);
                mg[2 * h] = dadd(0.0, a.x);  // (0 + o_0) + o_1, ssm.cpp:214-229
                mg[2 * h + 1] = dadd(0.0, a.y);
                if (p.x2) {
                    const double2 b2 = ldg2(p.x2 + src + 2 * h);
                    mg[2 * h] = dadd(mg[2 * h], b2.x);
                    mg[2 * h + 1] = dadd(mg[2 * h + 1], b2.y);
                }
                gg[2 * h] = g.x;
                gg[2 * h + 1] = g.y;
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) ap[k] = merge_approx(mg[k], gg[k]);
        }
        unsigned have = 0;  // bit k = v[k] holds the exact value
        if (dyn) {
            if (t == next_ref) {  // maybe_refresh
                in = 0;
                next_ref += p.n_refresh;
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) {  // detect_outliers, channel-local form
                if (!active || ((in >> k) & 1u)) continue;
                const float av = fabsf(ap[k].v);
                if (av * (1.0f - ap[k].eps) > thetaf * 1.0000003f) {
                    in |= 1u << k;
                } else if (av * (1.0f + ap[k].eps) >= thetaf * 0.9999997f) {
                    v[k] = merge_exact(mg[k], gg[k]);
                    have |= 1u << k;
                    if (fabs(v[k]) > theta) in |= 1u << k;
                }
            }
        }
        const double S = s_tab[t];
        const double inv = i_tab ? i_tab[t] : __ddiv_rn(1.0, S);
        if (active) {
            int c[CPT];
            const float invf = __double2float_rn(inv), capf = static_cast<float>(qa) + 1.0f;
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                c[k] = 0;
                if ((in >> k) & 1u) {
                    if (!((have >> k) & 1u)) v[k] = merge_exact(mg[k], gg[k]);
                    const double os = scale_from_peak(fabs(v[k]), qo);  // scale_for over the 1-value row
                    p.ocode[row * E + ch + k] = static_cast<int8_t>(static_cast<int>(quant_code_div(v[k], os, qo)));
                    p.oscale[row * E + ch + k] = os;
                } else {
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
                }
            }
            if constexpr (CPT == 4) {
                if (p.codes4)
                    *reinterpret_cast<uint16_t*>(p.codes4 + row * (E >> 1) + (ch >> 1)) = pack4(c[0], c[1], c[2], c[3]);
                else
                    *reinterpret_cast<char4*>(p.codes + row * E + ch) =
                        make_char4(static_cast<signed char>(c[0]), static_cast<signed char>(c[1]),
                                   static_cast<signed char>(c[2]), static_cast<signed char>(c[3]));
            } else {
                if (p.codes4)  // pack_int4: low nibble = even column
                    p.codes4[row * (E >> 1) + (ch >> 1)] = static_cast<uint8_t>((c[0] & 0xF) | ((c[1] & 0xF) << 4));
                else
                    *reinterpret_cast<char2*>(p.codes + row * E + ch) =
                        make_char2(static_cast<signed char>(c[0]), static_cast<signed char>(c[1]));
            }
        }
        // mask word of channels 32w..32w+31 from 32/CPT lanes x CPT bits (all zero in the common case)
        unsigned bits = active ? in << ((lane & (kLanesPerWord - 1)) * CPT) : 0u;
        if (__any_sync(0xffffffffu, bits != 0u)) {
#pragma unroll
            for (int o = kLanesPerWord / 2; o >= 1; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
        }
        if (active && (lane & (kLanesPerWord - 1)) == 0) {
            p.omask[row * J + (ch >> 5)] = bits;
            if (bits) atomicAdd(p.ocnt + row, __popc(bits));
        }
        if (ch == 0) p.s_row[row] = S;
    }
}

// Small batches (S x E within one warp per SM, e.g. C1 at batch 1): k1_channel's merge
// source with one lane per channel and one warp per (sample, refresh window, 32-channel
// group), the window's R tokens of o_0 / o_1 / gate loaded into registers at once (the
// four-channel kernel has a few dozen warps on the GPU at batch 1, each walking its
// tokens with one token's loads in flight). The mask word is the warp's ballot.
template <int R>
__global__ void __launch_bounds__(128) k1_merge_lane(const K1Params p) {
    const int E = p.E, T = p.T, J = E >> 5;
    const int lane = threadIdx.x & 31;
    const long gw = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int win = p.window, nwin = (T + win - 1) / win;
    if (gw >= static_cast<long>(p.S) * nwin * J) return;  // whole warps
    const int grp = static_cast<int>(gw % J);
    const long sw = gw / J;
    const int s = static_cast<int>(sw / nwin), wi = static_cast<int>(sw % nwin);
    const int t0 = wi * win, t1 = min(T, t0 + win);
    const int i = grp * 32 + lane;
    const bool dyn = p.mode == MODE_DYNAMIC;
    const double qa = qmax_for(p.abits), qo = qmax_for(p.obits);
    const int qai = static_cast<int>(qa);
    const double theta = p.cal.theta;
    const float thetaf = __double2float_rn(theta);
    const double* __restrict__ s_tab = dyn ? p.cal.s_in : p.cal.s_full;
    const double* __restrict__ i_tab = dyn ? p.inv_in : p.inv_full;
    int next_ref = (dyn && p.n_refresh > 0) ? t0 + p.n_refresh : 0x7fffffff;
    bool in = false;  // this channel is in O
    for (int c0 = t0; c0 < t1; c0 += R) {
        const int n = min(R, t1 - c0);
        double a0[R], a1[R], g[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            if (j < n) {
                const size_t src = (static_cast<size_t>(s) * T + row_at(p.order, c0 + j, T, p.grid)) * E + i;
                a0[j] = __ldg(p.x + src);
                a1[j] = p.x2 ? __ldg(p.x2 + src) : 0.0;
                g[j] = __ldg(p.gate + src);
            }
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
            if (j >= n) break;
            const int t = c0 + j;
            const size_t row = static_cast<size_t>(s) * T + t;
            double mg = dadd(0.0, a0[j]);  // (0 + o_0) + o_1, ssm.cpp:214-229
            if (p.x2) mg = dadd(mg, a1[j]);
            const MergeApprox ap = merge_approx(mg, g[j]);
            bool have = false;  // v holds the exact value
            double v = 0.0;
            if (dyn) {
                if (t == next_ref) {  // maybe_refresh
                    in = false;
                    next_ref += p.n_refresh;
                }
                if (!in) {  // detect_outliers, channel-local form
                    const float av = fabsf(ap.v);
                    if (av * (1.0f - ap.eps) > thetaf * 1.0000003f) {
                        in = true;
                    } else if (av * (1.0f + ap.eps) >= thetaf * 0.9999997f) {
                        v = merge_exact(mg, g[j]);
                        have = true;
                        in = fabs(v) > theta;
                    }
                }
            }
            const double S = s_tab[t];
            const double inv = i_tab ? i_tab[t] : __ddiv_rn(1.0, S);
            int c = 0;
            if (in) {
                if (!have) v = merge_exact(mg, g[j]);
                const double os = scale_from_peak(fabs(v), qo);  // scale_for over the 1-value row
                p.ocode[row * E + i] = static_cast<int8_t>(static_cast<int>(quant_code_div(v, os, qo)));
                p.oscale[row * E + i] = os;
            } else {
                // certified f32 quotient: |dq| <= (|q| + 1) (eps + 3 2^-24)
                const float capf = static_cast<float>(qa) + 1.0f;
                const float q = fminf(fmaxf(ap.v * __double2float_rn(inv), -capf), capf);
                const float r = rintf(q);
                if (!have && fabsf(q - r) < 0.5f - fmaf(fabsf(q) + 1.0f, ap.eps + 1.8e-7f, 1e-6f)) {
                    c = min(max(static_cast<int>(r), -qai), qai);
                } else {
                    if (!have) v = merge_exact(mg, g[j]);
                    c = quant_code_int(v, S, inv, qa, qai);
                }
            }
            if (p.codes4) {  // lanes 2k, 2k+1: one pack_int4 byte
                const unsigned nib = static_cast<unsigned>(c) & 0xFu;
                const unsigned hi = __shfl_down_sync(0xffffffffu, nib, 1);
                if (!(lane & 1)) p.codes4[row * (E >> 1) + (i >> 1)] = static_cast<uint8_t>(nib | (hi << 4));
            } else {
                p.codes[row * E + i] = static_cast<int8_t>(c);
            }
            const unsigned bits = __ballot_sync(0xffffffffu, in);
            if (lane == 0) {
                p.omask[row * J + grp] = bits;
                if (bits) atomicAdd(p.ocnt + row, __popc(bits));
                if (grp == 0) p.s_row[row] = S;
            }
        }
    }
}

// Staged fast path. Per CTA: one (sample, refresh window) of one direction, all
// E channels (blockDim = E/4 rounded to warps). Rows of `rc` steps per stage,
// kK1Stages stages: chunk c lands in stage c % kK1Stages by per-row bulk copies
// on an mbarrier; chunk c + kK1Stages is issued once every thread has finished
// chunk c. 24 KB stages
// (rc = 4 rows at E = 768; 4 CTAs per SM, register-limited): x_proj pair / in_proj
// 147 / 105 us; 20 KB (rc = 3) 152 / 112 us; 32 KB (3 CTAs) was slower still.
constexpr int kK1StageBytes = 24 * 1024;
constexpr int kK1Stages = 2;  // 3 stages (fewer CTAs per SM) measured 165 / 117 us vs 155 / 113
constexpr int kK1MaxRc = 16;
constexpr int kK1MaxWin = 64;  // windows up to 64 steps keep their scales in shared memory
struct K1Dirs {
    K1Params p[2];
    int n = 1;       // directions in this launch
    int mirror = 0;  // direction 1 runs window nwin-1-w (row-reverse of direction 0): same rows, same time
    int rc = 1;      // steps per stage
};

__device__ __forceinline__ int k1_row_of(const K1Params& p, int t) {
    return row_at(p.order, t, p.T, p.grid);
}

// the outlier channels of a quad: own scale |x|/q_o, code at o_bits (out of line: rare)
__device__ __noinline__ void outliers4(unsigned in, double v0, double v1, double v2, double v3, double qo,
                                       int8_t* ocode, double* oscale) {
    const double v[4] = {v0, v1, v2, v3};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if ((in >> k) & 1u) {
            const double os = scale_from_peak(fabs(v[k]), qo);  // scale_for over the 1-value row
            ocode[k] = static_cast<int8_t>(static_cast<int>(quant_code_div(v[k], os, qo)));
            oscale[k] = os;
        }
    }
}

template <int SRC, bool PK>
__global__ void __launch_bounds__(256) k1_staged(const __grid_constant__ K1Dirs dirs) {
    extern __shared__ __align__(128) unsigned char k1_smem[];
    double* stage = reinterpret_cast<double*>(k1_smem);  // [kK1Stages][rc][E]
    __shared__ uint64_t bar[kK1Stages];
    __shared__ int cnt[kK1Stages][kK1MaxRc];     // |O(t)| of the chunk's rows
    __shared__ double rsv[kK1Stages][kK1MaxRc];  // D1 row factors of the chunk's rows
    __shared__ double2 si_win[kK1MaxWin];         // {S^I(t), 1/S^I(t)} of the window's steps
    const int d = dirs.n == 2 ? static_cast<int>(blockIdx.y & 1) : 0;
    const K1Params& p = dirs.p[d];
    const int yy = dirs.n == 2 ? static_cast<int>(blockIdx.y >> 1) : static_cast<int>(blockIdx.y);
    const int E = p.E, T = p.T, J = E >> 5, rc = dirs.rc;
    const int win = p.window, nwin = (T + win - 1) / win;
    const int s = yy / nwin;
    int wi = yy % nwin;
    if (d == 1 && dirs.mirror) wi = nwin - 1 - wi;
    const int t0 = wi * win, t1 = min(T, t0 + win);
    const int nchunks = (t1 - t0 + rc - 1) / rc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int ch = tid * 4;
    const bool active = ch < E;
    const uint32_t row_bytes = static_cast<uint32_t>(E) * 8u;

    auto issue = [&](int c) {  // thread 0
        const int buf = c % kK1Stages, ts = t0 + c * rc, te = min(t1, ts + rc);
        ptx::mbar_arrive_expect_tx(&bar[buf], static_cast<uint32_t>(te - ts) * row_bytes);
        for (int t = ts; t < te; ++t)
            ptx::bulk_g2s(stage + (static_cast<size_t>(buf) * rc + (t - ts)) * E,
                     p.x + (static_cast<size_t>(s) * T + k1_row_of(p, t)) * E, row_bytes, &bar[buf]);
    };
    if (tid == 0) {  // the first chunks are in flight before the CTA barrier
        for (int b = 0; b < kK1Stages; ++b) ptx::mbar_init(&bar[b], 1);
        ptx::fence_barrier_init();
        for (int c = 0; c < kK1Stages && c < nchunks; ++c) issue(c);
    }
    for (int i = tid; i < kK1Stages * kK1MaxRc; i += blockDim.x) cnt[i / kK1MaxRc][i % kK1MaxRc] = 0;
    {
        const bool dyn0 = p.mode == MODE_DYNAMIC;
        const double* st = dyn0 ? p.cal.s_in : p.cal.s_full;
        const double* it = dyn0 ? p.inv_in : p.inv_full;
        for (int i = tid; i < t1 - t0 && i < kK1MaxWin; i += blockDim.x) {
            const double S = st[t0 + i];
            si_win[i] = make_double2(S, it ? it[t0 + i] : __ddiv_rn(1.0, S));
        }
    }
    __syncthreads();

    // every field the loop needs, read once (the direction's parameter block is
    // selected at run time)
    const bool dyn = p.mode == MODE_DYNAMIC;
    const int n_refresh = p.n_refresh;
    const double qa = qmax_for(p.abits), qo = qmax_for(p.obits);
    const int qai = static_cast<int>(qa);
    const double theta = p.cal.theta;
    const double* __restrict__ s_tab = dyn ? p.cal.s_in : p.cal.s_full;
    const double* __restrict__ i_tab = dyn ? p.inv_in : p.inv_full;
    int8_t* __restrict__ const codes = p.codes;
    uint8_t* __restrict__ const codes4 = p.codes4;  // PK (a template flag: the int8 form keeps its 76 registers)
    int8_t* __restrict__ const ocode = p.ocode;
    double* __restrict__ const oscale = p.oscale;
    uint32_t* __restrict__ const omask = p.omask;
    double* __restrict__ const s_row = p.s_row;
    int* __restrict__ const ocnt = p.ocnt;
    const unsigned qq = (static_cast<unsigned>(qai) << 16) | static_cast<unsigned>(qai);
    const unsigned nq = (static_cast<unsigned>(-qai) << 16) | (static_cast<unsigned>(-qai) & 0xFFFFu);
    int next_ref = (dyn && n_refresh > 0) ? t0 + n_refresh : 0x7fffffff;
    unsigned in = 0;  // bit k: channel ch+k is in O
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c % kK1Stages, ts = t0 + c * rc, te = min(t1, ts + rc);
        const double* sb = stage + static_cast<size_t>(buf) * rc * E;
        ptx::mbar_wait(&bar[buf], static_cast<uint32_t>((c / kK1Stages) & 1));
        if (SRC == K1_SRC_RMSNORM) {
            // 1/sqrt(mean(x^2) + 1e-6): 32 lane-strided partials (channel k -> partial
            // k%32, k ascending) combined by an xor butterfly (oracle/driver.hpp rmsnorm_row)
            for (int r = warp; r < te - ts; r += nwarps) {
                const double* xr = sb + static_cast<size_t>(r) * E;
                double ps = 0.0;
                for (int k = lane; k < E; k += 32) ps = dadd(ps, dmul(xr[k], xr[k]));
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) ps = dadd(ps, __shfl_xor_sync(0xffffffffu, ps, o));
                if (lane == 0) rsv[buf][r] = __ddiv_rn(1.0, __dsqrt_rn(dadd(__ddiv_rn(ps, static_cast<double>(E)), 1e-6)));
            }
            __syncthreads();
        }
        // running pointers (row = s*T + t; the staged row `slot` of this chunk)
        const double* xr = sb + ch;
        const size_t row0 = static_cast<size_t>(s) * T + ts;
        int8_t* cp = PK ? nullptr : codes + row0 * E + ch;
        uint16_t* cp4 = PK ? reinterpret_cast<uint16_t*>(codes4 + row0 * (E >> 1) + (ch >> 1)) : nullptr;
        uint32_t* mp = omask + row0 * J + (ch >> 5);
        for (int t = ts; t < te; ++t, xr += E, mp += J, cp += (PK ? 0 : E), cp4 += (PK ? (E >> 2) : 0)) {
            const int slot = t - ts;
            const size_t row = row0 + slot;
            double S, inv;
            if (t - t0 < kK1MaxWin) {
                const double2 si = si_win[t - t0];
                S = si.x;
                inv = si.y;
            } else {
                S = s_tab[t];
                inv = i_tab ? i_tab[t] : __ddiv_rn(1.0, S);
            }
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            if (active) {
                const double2 lo = *reinterpret_cast<const double2*>(xr);
                const double2 hi = *reinterpret_cast<const double2*>(xr + 2);
                v[0] = lo.x;
                v[1] = lo.y;
                v[2] = hi.x;
                v[3] = hi.y;
                if (SRC == K1_SRC_RMSNORM) {
                    const double r = rsv[buf][slot];
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[k] = dmul(v[k], r);
                }
            }
            if (dyn) {
                if (t == next_ref) {  // maybe_refresh
                    in = 0;
                    next_ref += n_refresh;
                }
                // detect_outliers, channel-local form (one predicate chain; the bits only
                // when a channel crosses theta)
                if (any_abs_gt4(v[0], v[1], v[2], v[3], theta))
                    in |= (fabs(v[0]) > theta ? 1u : 0u) | (fabs(v[1]) > theta ? 2u : 0u) |
                          (fabs(v[2]) > theta ? 4u : 0u) | (fabs(v[3]) > theta ? 8u : 0u);
            }
            // inlier codes for all four channels: tq = fl(v * inv + 1.5 * 2^52) holds
            // RNE(v * inv) in its low word while |v * inv| < 2^31 and d = fl(v * inv - that)
            // is its distance, so quant_code_int's test reads |d| <= 0.4999999999990 (a NaN
            // fails it); the integer clamp replaces its f64 clamp. In dynamic mode inliers
            // have |v| <= theta, so theta / S < 2^14 bounds every inlier quotient of the row
            // (outlier channels' codes are zeroed); otherwise each quotient is range-checked
            // (|q| < 2^14 also keeps the s16x2 clamp exact). A failed test decides the four
            // exactly (quant_code_int).
            constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
            int cc[4];
            bool tie = false;
            auto codes_of = [&](auto ranged) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double tq = __fma_rn(v[k], inv, kMagic);
                    const double r = dadd(tq, -kMagic);
                    cc[k] = __double2loint(tq);
                    tie |= !(fabs(__fma_rn(v[k], inv, -r)) <= 0.4999999999990);
                    if constexpr (decltype(ranged)::value) tie |= !(fabs(r) < 16384.0);
                }
            };
            if (dyn && theta * inv < 16384.0)
                codes_of(std::false_type{});
            else
                codes_of(std::true_type{});
            if (tie) {
#pragma unroll
                for (int k = 0; k < 4; ++k) cc[k] = quant_code_int(v[k], S, inv, qa, qai);
            }
            if (active) {
                // clamp as two s16x2 pairs, bytes c0..c3
                const unsigned p01 = __vmaxs2(__vmins2(__byte_perm(cc[0], cc[1], 0x5410), qq), nq);
                const unsigned p23 = __vmaxs2(__vmins2(__byte_perm(cc[2], cc[3], 0x5410), qq), nq);
                unsigned w = __byte_perm(p01, p23, 0x6420);
                if (in) {
                    w &= ~(((in * 0x00204081u) & 0x01010101u) * 0xFFu);  // outlier channels: code 0
                    outliers4(in, v[0], v[1], v[2], v[3], qo, ocode + row * E + ch, oscale + row * E + ch);
                }
                if constexpr (PK) {
                    const unsigned n = w & 0x0F0F0F0Fu;  // pack_int4: low nibble = even column
                    *cp4 = static_cast<uint16_t>(__byte_perm(n | (n >> 4), 0u, 0x0020));
                } else {
                    *reinterpret_cast<unsigned*>(cp) = w;
                }
            }
            // mask word of channels 32w..32w+31 from 8 lanes x 4 bits (all zero in the common case)
            unsigned bits = active ? in << ((lane & 7) * 4) : 0u;
            if (__any_sync(0xffffffffu, bits != 0u)) {
#pragma unroll
                for (int o = 4; o >= 1; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
                if (active && (lane & 7) == 0 && bits) atomicAdd(&cnt[buf][slot], __popc(bits));
            }
            if (active && (lane & 7) == 0) *mp = bits;
            if (tid == 0) s_row[row] = S;
        }
        __syncthreads();  // stage `buf` consumed, counts complete
        if (tid < te - ts) {
            ocnt[static_cast<size_t>(s) * T + ts + tid] = cnt[buf][tid];
            cnt[buf][tid] = 0;
        }
        if (tid == 0 && c + kK1Stages < nchunks) {
            ptx::fence_async_smem();  // generic-proxy reads of the stage before the async refill
            issue(c + kK1Stages);
        }
    }
}

// Register-resident window path (plain / RMSNorm sources, E % 64 == 0): a CTA owns
// one (sample, refresh window) of one direction with blockDim = E/2, one thread
// per channel pair; a chunk of R rows of the window (R >= the window in the usual
// case) is loaded into registers at once (R x 16 B per thread in flight, like the
// conv's), and the channel-local detector runs down the rows with the channel
// state in a register. Each thread's two codes are independent of every other
// thread's, so the only CTA-wide work is D1's row factor (squares through shared
// memory, one warp per row in the k%32 partial order of rmsnorm_row) and |O(t)|.
__device__ __forceinline__ bool any_abs_gt2(double a, double b, double th) {
    unsigned r;
    asm("{\n\t.reg .pred p;\n\t.reg .f64 x;\n\t"
        "abs.f64 x, %1;\n\tsetp.gt.f64 p, x, %3;\n\t"
        "abs.f64 x, %2;\n\tsetp.gt.or.f64 p, x, %3, p;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r) : "d"(a), "d"(b), "d"(th));
    return r != 0u;
}

// the rare paths out of line, so the unrolled rows stay compact in the icache
__device__ __noinline__ int2 codes_exact2(double v0, double v1, double S, double inv, double qa, int qai) {
    return make_int2(quant_code_int(v0, S, inv, qa, qai), quant_code_int(v1, S, inv, qa, qai));
}
__device__ __noinline__ void outliers2(unsigned in, double v0, double v1, double qo, int8_t* ocode, double* oscale) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if ((in >> k) & 1u) {
            const double v = k ? v1 : v0;
            const double os = scale_from_peak(fabs(v), qo);  // scale_for over the 1-value row
            ocode[k] = static_cast<int8_t>(static_cast<int>(quant_code_div(v, os, qo)));
            oscale[k] = os;
        }
    }
}

template <int SRC, bool PK, int R>
__global__ void __launch_bounds__(384, 2) k1_window(const __grid_constant__ K1Dirs dirs) {
    extern __shared__ __align__(16) double k1w_sq[];  // RMSNorm: [R][E] squares
    __shared__ int cnt[R];
    __shared__ double rsv[R], s_s[R], s_i[R];
    const int d = dirs.n == 2 ? static_cast<int>(blockIdx.x & 1) : 0;
    const K1Params& p = dirs.p[d];
    const int yy = dirs.n == 2 ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int E = p.E, T = p.T, J = E >> 5;
    const int win = p.window, nwin = (T + win - 1) / win;
    const int s = yy / nwin;
    int wi = yy % nwin;
    if (d == 1 && dirs.mirror) wi = nwin - 1 - wi;
    const int t0 = wi * win, t1 = min(T, t0 + win);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int ch = tid * 2;
    const bool dyn = p.mode == MODE_DYNAMIC;
    const int n_refresh = p.n_refresh;
    const double qa = qmax_for(p.abits), qo = qmax_for(p.obits);
    const int qai = static_cast<int>(qa);
    const double theta = p.cal.theta;
    const double* __restrict__ s_tab = dyn ? p.cal.s_in : p.cal.s_full;
    const double* __restrict__ i_tab = dyn ? p.inv_in : p.inv_full;
    const double* __restrict__ xs = p.x + static_cast<size_t>(s) * T * E + ch;
    const unsigned qq = (static_cast<unsigned>(qai) << 16) | static_cast<unsigned>(qai);
    const unsigned nq = (static_cast<unsigned>(-qai) << 16) | (static_cast<unsigned>(-qai) & 0xFFFFu);
    int next_ref = (dyn && n_refresh > 0) ? t0 + n_refresh : 0x7fffffff;
    unsigned in = 0;  // bit k: channel ch+k is in O
    if (tid < R) cnt[tid] = 0;
    for (int c0 = t0; c0 < t1; c0 += R) {
        const int n = min(R, t1 - c0);
        double2 xv[R];
        if (p.order <= 1) {  // identity / reversed order: rows at a fixed stride
            const long long step = p.order == 1 ? -static_cast<long long>(E) : static_cast<long long>(E);
            const double* b = xs + static_cast<size_t>(p.order == 1 ? T - 1 - c0 : c0) * E;
#pragma unroll
            for (int j = 0; j < R; ++j)
                if (j < n) xv[j] = ldg2(b + j * step);
        } else {
#pragma unroll
            for (int j = 0; j < R; ++j)
                if (j < n) xv[j] = ldg2(xs + static_cast<size_t>(k1_row_of(p, c0 + j)) * E);
        }
        if (tid < n) {
            const double S = s_tab[c0 + tid];
            s_s[tid] = S;
            s_i[tid] = i_tab ? i_tab[c0 + tid] : __ddiv_rn(1.0, S);
        }
        if (SRC == K1_SRC_RMSNORM) {
            // 1/sqrt(mean(x^2) + 1e-6): 32 lane-strided partials (channel k -> partial
            // k%32, k ascending) combined by an xor butterfly (oracle/driver.hpp rmsnorm_row)
#pragma unroll
            for (int j = 0; j < R; ++j)
                if (j < n)
                    *reinterpret_cast<double2*>(k1w_sq + static_cast<size_t>(j) * E + ch) =
                        make_double2(dmul(xv[j].x, xv[j].x), dmul(xv[j].y, xv[j].y));
            __syncthreads();
            for (int r = warp; r < n; r += nwarps) {
                const double* q = k1w_sq + static_cast<size_t>(r) * E;
                double ps = 0.0;
                for (int k = lane; k < E; k += 32) ps = dadd(ps, q[k]);
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) ps = dadd(ps, __shfl_xor_sync(0xffffffffu, ps, o));
                if (lane == 0) rsv[r] = __ddiv_rn(1.0, __dsqrt_rn(dadd(__ddiv_rn(ps, static_cast<double>(E)), 1e-6)));
            }
        }
        __syncthreads();  // row scales, D1 factors, zeroed counts
#pragma unroll
        for (int j = 0; j < R; ++j) {
            if (j >= n) break;
            const int t = c0 + j;
            const size_t row = static_cast<size_t>(s) * T + t;
            const double S = s_s[j], inv = s_i[j];
            double v0 = xv[j].x, v1 = xv[j].y;
            if (SRC == K1_SRC_RMSNORM) {
                const double r = rsv[j];
                v0 = dmul(v0, r);
                v1 = dmul(v1, r);
            }
            if (dyn) {
                if (t == next_ref) {  // maybe_refresh
                    in = 0;
                    next_ref += n_refresh;
                }
                if (any_abs_gt2(v0, v1, theta))  // detect_outliers, channel-local form
                    in |= (fabs(v0) > theta ? 1u : 0u) | (fabs(v1) > theta ? 2u : 0u);
            }
            // k1_staged's code test on two channels (tq = fl(v * inv + 1.5 * 2^52), d the
            // remainder; quotients bounded by theta / S in dynamic mode, else range-checked)
            constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
            const double tq0 = __fma_rn(v0, inv, kMagic), tq1 = __fma_rn(v1, inv, kMagic);
            const double r0 = dadd(tq0, -kMagic), r1 = dadd(tq1, -kMagic);
            int c0i = __double2loint(tq0), c1i = __double2loint(tq1);
            bool tie = !(fabs(__fma_rn(v0, inv, -r0)) <= 0.4999999999990) |
                       !(fabs(__fma_rn(v1, inv, -r1)) <= 0.4999999999990);
            if (!(dyn && theta * inv < 16384.0)) tie |= !(fabs(r0) < 16384.0) | !(fabs(r1) < 16384.0);
            if (tie) {
                const int2 c = codes_exact2(v0, v1, S, inv, qa, qai);
                c0i = c.x;
                c1i = c.y;
            }
            unsigned pr = __vmaxs2(__vmins2(__byte_perm(c0i, c1i, 0x5410), qq), nq);  // s16 x2
            if (in) {
                pr &= ~(((in & 1u) ? 0x0000FFFFu : 0u) | ((in & 2u) ? 0xFFFF0000u : 0u));  // outliers: code 0
                outliers2(in, v0, v1, qo, p.ocode + row * E + ch, p.oscale + row * E + ch);
            }
            if constexpr (PK)  // pack_int4: low nibble = even column
                p.codes4[row * (E >> 1) + tid] = static_cast<uint8_t>((pr & 0xFu) | ((pr >> 12) & 0xF0u));
            else
                *reinterpret_cast<uint16_t*>(p.codes + row * E + ch) = static_cast<uint16_t>(__byte_perm(pr, 0u, 0x0020));
            // mask word of channels 32w..32w+31 from 16 lanes x 2 bits (all zero in the common case)
            unsigned bits = in << ((lane & 15) * 2);
            if (__any_sync(0xffffffffu, bits != 0u)) {
#pragma unroll
                for (int o = 8; o >= 1; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
                if ((lane & 15) == 0 && bits) atomicAdd(&cnt[j], __popc(bits));
            }
            if ((lane & 15) == 0) p.omask[row * J + (ch >> 5)] = bits;
            if (tid == 0) p.s_row[row] = S;
        }
        __syncthreads();  // counts complete, s_s / s_i / rsv / squares consumed
        if (tid < n) {
            p.ocnt[static_cast<size_t>(s) * T + c0 + tid] = cnt[tid];
            cnt[tid] = 0;
        }
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
        const int crow = row_at(p.order, t, p.T, p.grid);
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
            int ci = 0;
            if (valid) {
                double c = 0.0;
                if (isout) {
                    const double os = scale_from_peak(fabs(v[j]), qo);
                    p.ocode[row * E + ch] = static_cast<int8_t>(static_cast<int>(quant_code_div(v[j], os, qo)));
                    p.oscale[row * E + ch] = os;
                } else {
                    c = quant_code_inv(v[j], S, inv, qa);
                }
                ci = static_cast<int>(c);
                if (!p.codes4) p.codes[row * E + ch] = static_cast<int8_t>(ci);
            }
            if (p.codes4) {  // lanes 2i, 2i+1 hold channels 32j + 2i, 32j + 2i + 1: one packed byte
                const unsigned nib = static_cast<unsigned>(ci) & 0xFu;
                const unsigned hi = __shfl_down_sync(0xffffffffu, nib, 1);
                if (valid && !(lane & 1)) p.codes4[row * (E >> 1) + (ch >> 1)] = static_cast<uint8_t>(nib | (hi << 4));
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
    const int nwin = (p.T + p.window - 1) / p.window;
    if (static_cast<long>(p.S) * p.E <= 148L * 32) {  // small batches: a lane per channel
        const long warps = static_cast<long>(p.S) * nwin * (p.E / 32);
        const unsigned blocks = static_cast<unsigned>((warps * 32 + 127) / 128);
        if (p.window <= 10) k1_merge_lane<10><<<blocks, 128, 0, st>>>(p);
        else k1_merge_lane<16><<<blocks, 128, 0, st>>>(p);
        ++kernel_launch_counter();
        return cudaGetLastError();
    }
    constexpr int kCpt = K1_MERGE_CPT;
    const int units = p.E / kCpt, threads = units >= 256 ? 256 : ((units + 31) / 32) * 32;
    dim3 grid((units + threads - 1) / threads, p.S * nwin);
    k1_channel<SRC, kCpt><<<grid, threads, 0, st>>>(p);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

template <int SRC, bool PK>
static cudaError_t launch_staged_pk(const K1Dirs& dirs, cudaStream_t st) {
    const K1Params& p = dirs.p[0];
    const int nwin = (p.T + p.window - 1) / p.window;
    const int threads = ((p.E / 4 + 31) / 32) * 32;  // E <= 1024: one CTA covers every channel
    const size_t smem = static_cast<size_t>(kK1Stages) * dirs.rc * p.E * sizeof(double);
    cudaError_t e = ensure_smem_attr<k1_staged<SRC, PK>>(static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k1_staged<SRC, PK><<<dim3(1, p.S * nwin * dirs.n), threads, smem, st>>>(dirs);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

template <int SRC, bool PK, int R>
static cudaError_t launch_window_r(const K1Dirs& dirs, cudaStream_t st) {
    const K1Params& p = dirs.p[0];
    const int nwin = (p.T + p.window - 1) / p.window;
    const size_t smem = SRC == K1_SRC_RMSNORM ? static_cast<size_t>(R) * p.E * sizeof(double) : 0;
    cudaError_t e = ensure_smem_attr<k1_window<SRC, PK, R>>(static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    k1_window<SRC, PK, R><<<p.S * nwin * dirs.n, p.E / 2, smem, st>>>(dirs);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

template <int SRC, bool PK>
static cudaError_t launch_window(const K1Dirs& dirs, cudaStream_t st) {
    // rows per register chunk: the whole window when it has <= 12 rows, else 12
    const int w = dirs.p[0].window;
    if (w <= 8) return launch_window_r<SRC, PK, 8>(dirs, st);
    if (w <= 10) return launch_window_r<SRC, PK, 10>(dirs, st);
    return launch_window_r<SRC, PK, 12>(dirs, st);
}

template <int SRC>
static cudaError_t launch_staged(const K1Dirs& dirs, cudaStream_t st) {
    if ((dirs.p[0].codes4 != nullptr) != (dirs.p[1].codes4 != nullptr)) return cudaErrorInvalidValue;
    // the register window kernel on request, and for small batches (S x E within one warp
    // per SM: C1 12.6 / 12.3 vs 14.3 / 13.4 us for the in_proj / x_proj pair inputs)
    const bool small = static_cast<long>(dirs.p[0].S) * dirs.p[0].E <= 148L * 32;
    if ((dirs.p[0].window_kernel || small) && dirs.p[0].E % 64 == 0 && dirs.p[0].E <= 768)
        return dirs.p[0].codes4 ? launch_window<SRC, true>(dirs, st) : launch_window<SRC, false>(dirs, st);
    return dirs.p[0].codes4 ? launch_staged_pk<SRC, true>(dirs, st) : launch_staged_pk<SRC, false>(dirs, st);
}

static K1Dirs k1_dirs(const K1Params* ps, int n) {
    K1Dirs d;
    d.n = n;
    d.p[0] = ps[0];
    d.p[1] = n > 1 ? ps[1] : ps[0];
    d.mirror = n > 1 && ps[0].order <= 0 && ps[1].order == 1;
    // stage rows: 24 KB stages, but no more shared memory per CTA than the CTAs the
    // registers allow can share (narrow E: more, smaller CTAs per SM; E = 384: 4 rows
    // instead of 8, 8 CTAs per SM instead of 4)
    const int threads = ((ps[0].E / 4 + 31) / 32) * 32;
    const int ctas = std::max(1, 65536 / (80 * threads));
    const int rows_smem = (220 * 1024 / ctas) / (kK1Stages * ps[0].E * 8);
    const int rows = std::min(kK1StageBytes / (ps[0].E * 8), rows_smem);
    d.rc = std::max(1, std::min({rows, kK1MaxRc, ps[0].window}));
    return d;
}

static bool k1_fast(const K1Params& p) {
    // the channel-parallel kernels need: a quantizing mode, no DetectResult output,
    // the channel-local detector exact (no literal steps) and E % 32 == 0
    return p.mode != MODE_FP && !p.scanned && !p.force_literal && (p.E % 32) == 0;
}

cudaError_t launch_k1(const K1Params& p, cudaStream_t st) {
    if (p.E < 1 || p.E > 1024 || p.T < 1 || p.S < 1 || p.window < 1) return cudaErrorInvalidValue;
    if (p.codes4 && (p.abits != 4 || (p.E & 1))) return cudaErrorInvalidValue;  // nibbles hold [-7, 7]
    if (!p.codes4 && !p.codes && p.mode != MODE_FP) return cudaErrorInvalidValue;
    const bool fast = k1_fast(p);
    switch (p.src) {
        case K1_SRC_PLAIN: return fast ? launch_staged<K1_SRC_PLAIN>(k1_dirs(&p, 1), st) : launch_literal<K1_SRC_PLAIN>(p, st);
        case K1_SRC_RMSNORM:
            return fast ? launch_staged<K1_SRC_RMSNORM>(k1_dirs(&p, 1), st) : launch_literal<K1_SRC_RMSNORM>(p, st);
        case K1_SRC_MERGE: return fast ? launch_channel<K1_SRC_MERGE>(p, st) : launch_literal<K1_SRC_MERGE>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k1_dirs(const K1Params* ps, int n, cudaStream_t st) {
    // one staged launch when every direction quantizes the same plain rows on the fast path
    bool pair = n == 2;
    for (int i = 0; pair && i < n; ++i)
        pair = ps[i].src == K1_SRC_PLAIN && k1_fast(ps[i]) && ps[i].x == ps[0].x && ps[i].S == ps[0].S &&
               ps[i].T == ps[0].T && ps[i].E == ps[0].E && ps[i].window == ps[0].window && ps[i].E <= 1024 &&
               ps[i].E >= 1;
    if (pair) return launch_staged<K1_SRC_PLAIN>(k1_dirs(ps, n), st);
    for (int i = 0; i < n; ++i) {
        const cudaError_t e = launch_k1(ps[i], st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace ob
