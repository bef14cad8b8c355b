// K3 fast path: quantized S6 selective scan for the dynamic / static modes
// where the channel-local detector is exact, both scan
// directions in one launch.
//
// Work split. A CTA owns 32 channels of one (sample, direction) (small CTAs
// keep the last wave's tail short: 8 of them share an SM); two adjacent lanes
// own one channel, 8 of its N = 16 states each, so a warp covers 16 channels. Warps are independent: each stages its own copy of the
// per-step values in its own shared-memory slice and synchronises only with
// __syncwarp, so a warp delayed by a rare exact fallback never stalls the
// others. The two halves of a channel exchange two values per step through
// shuffles: the h peak (max is order-free) and the running output sum —
// the first half computes 0 + C_0 h_0 + ... + C_7 h_7 in order and the second
// half continues the same chain with C_8 h_8 ... C_15 h_15, which is the
// reference's sequential sum (ssm.cpp:170-174) bit-for-bit.
//
// Steps are processed in chunks of 8. Everything that does not depend on the
// carried state is computed for the whole chunk first, with the chunk's steps
// as independent instruction streams, and staged in the warp's shared memory: per step
// B, C and the calibrated scales; per channel x = dpre + b_delta (exact), an
// f32 delta = softplus(x) with its proven relative error bound, and u.
//
// Exactness (the reference values are f64, quant.cpp:29-35). Every code,
// detector decision and dequantized value equals the reference's:
//  * detector peaks: a_bar > 0 and delta >= 0, so max_m a_bar = exp(fl(delta*
//    Amax)) and max_m |b_bar| = fl(delta*max_m|B_m|) (monotone rounding). Both
//    are evaluated in f32 with error bounds; a decision within the bound of
//    theta, an outlier channel's scale and every fallback below use the exact
//    f64 delta = softplus(x), exp and IEEE quotients;
//  * a_bar and b_bar codes: q = x / s in f32 (ex2.approx for the exp) with a
//    proven relative error bound; round(q) is used when q is farther than that
//    bound from a half-integer, else the element is recomputed in f64 (rare).
//    Dequantized values are code * s in f64, as fake_quant_step's;
//  * h update (f64, reference order), h codes certified the same way from the
//    f32 rounding of the exact h (the f32 peak equals fl32 of the exact peak),
//    the output sum in the reference's order.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "merge_f32.cuh"
#include "scan_f32.cuh"
#include "sm100_ptx.cuh"

#include <type_traits>

namespace ob {

constexpr int kCh = 32;        // channels per CTA
constexpr int kThr = 2 * kCh;  // two threads per channel
constexpr int kChunk = 8;      // steps staged per chunk

struct ScanDirs {
    ScanParams d[2];
    int n = 1;              // directions in this launch
    // the out_proj input K1 fused into the one-thread-per-channel kernel (merge_tail):
    // the last of the n directions to finish a (sample, 32-channel group) quantizes it
    K1Params merge;
    int* merge_cnt = nullptr;  // [S][E/32] finish counters (zero between launches)
};

struct __align__(16) StepShared {
    double B[16], C[16];
    double Sa, Sb, Sh, Bmax;
    float BSf[16];  // f32(B_m) * f32(1/S_b): the inlier b_bar quotient per unit delta
    float invSaf, invSbf, invShf, Bmaxf;
    float LA;  // ln2 * (1 + max(0, log2(1/S_a))): bound of ln2*|log2 a_bar| where inlier rounding matters
    float BSmaxf;  // max_m |BSf[m]|: no b_bar quotient of a channel exceeds delta * BSmaxf
    float hA0, hA1;  // inlier a_bar certification margin = hA0 - hA1 * eps_delta (see the step loop)
    int keep;        // outlier flags kept at this step: 0 at a maybe_refresh point (quant.cpp:303-311), else ~0
    int ocol;        // crow * E: canonical token of this scan step (ssm.cpp:30-46), as an output offset
    int pad[2];
    float Saf, Sbf, Shf;  // f32(S_a), f32(S_b), f32(S_h): the f32 state update of k3_scan_c1<FS>
    float pad2;
};

static_assert(sizeof(StepShared) % 16 == 0, "bulk-copied step tables");
constexpr int kWarpCh = 16;  // channels per warp
// Per-warp slice: step tables and raw per-channel inputs are double-buffered
// (chunk k+1 is in flight while chunk k is scanned); x / deltaf / epsd hold
// the current chunk.
// The exact f64 transcendental values (glibc's algorithms) are needed only on the
// rare exact paths: out of line, so the certified f32 loop keeps its code size.
__device__ __noinline__ double exp_call(double x) { return gl::exp(x); }
__device__ __noinline__ double softplus_call(double x) { return softplus_d(x); }
__device__ __noinline__ double qdiv_call(double x, double sc, double q) { return quant_code_div(x, sc, q); }
// outlier-channel scale and its reciprocal (rare: a channel's first outlier step)
__device__ __noinline__ double scale_call(double peak, double q) { return scale_from_peak(peak, q); }
__device__ __noinline__ double recip_call(double x) { return __ddiv_rn(1.0, x); }

struct WarpSmem {
    StepShared st[2][kChunk];
    double dp[2][kChunk][kWarpCh];  // x_proj delta pre-activations (raw)
    double u[2][kChunk][kWarpCh];
    double x[kChunk][kWarpCh];      // dpre + b_delta, exact (softplus on demand)
    float deltaf[kChunk][kWarpCh];  // f32 softplus(x)
    float epsd[kChunk][kWarpCh];    // relative error bound of deltaf
    uint64_t bar[2];
};


// Round to nearest via the magic 1.5*2^23: the f32 bit pattern of q + 1.5*2^23 is
// 0x4B400000 + code. Integer -> f64 avoids the conversion pipe (I2F.F64 measured
// 1.7x slower here): a_bar codes (>= 0) go under the exponent of 2^52 into one
// DFMA; b_bar and h codes use F2F.F64.F32 of the exact f32 integer, which
// balances the XU against the FP64/ALU issue slots.
constexpr unsigned kMagicBits = 0x4B400000u;
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(ptx::smem_u32(dst)), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}

// Per (direction, sample, scan step) tables the scan consumes: B, C, the
// calibrated scales and their f32 inverses / copies, the b_bar quotients per unit
// delta and max_m |B_m|. One warp per (direction, step, group of kTabSamples
// samples): the step's calibration fields (global loads of the scale tables, a
// log2) are computed once and kept in the warp's shared record, then each sample
// overwrites its B / C fields (lane j holds column E + j of the x_proj row; all the
// group's rows are loaded at once) and the record leaves as 16-byte coalesced chunks.
constexpr int kTabSamples = 8;
__global__ void __launch_bounds__(256) k3_step_tables(const ScanDirs P, int ndirs, StepShared* __restrict__ out) {
    __shared__ StepShared rec[8];
    const int wi = threadIdx.x >> 5, gw = blockIdx.x * 8 + wi, lane = threadIdx.x & 31;
    const ScanParams& p0 = P.d[0];
    const int S = p0.S, T = p0.T, groups = (S + kTabSamples - 1) / kTabSamples;
    if (gw >= ndirs * T * groups) return;
    const int dd = gw / (T * groups), rem = gw - dd * T * groups, t = rem / groups, s0 = (rem % groups) * kTabSamples;
    const ScanParams& p = P.d[dd];
    const bool dyn = p.mode == MODE_DYNAMIC;
    StepShared& ss = rec[wi];
    const double Sb = dyn ? p.cal[1].s_in[t] : p.cal[1].s_full[t];
    const double* ib = dyn ? p.cal[1].inv_in : p.cal[1].inv_full;
    const float invSbf = __double2float_rn(ib ? ib[t] : __ddiv_rn(1.0, Sb));
    if (lane == 0) {
        const double Sa = dyn ? p.cal[0].s_in[t] : p.cal[0].s_full[t];
        const double Sh = dyn ? p.cal[2].s_in[t] : p.cal[2].s_full[t];
        const double* ia = dyn ? p.cal[0].inv_in : p.cal[0].inv_full;
        const double* ih = dyn ? p.cal[2].inv_in : p.cal[2].inv_full;
        ss.Sa = Sa;
        ss.Sb = Sb;
        ss.Sh = Sh;
        ss.invSaf = __double2float_rn(ia ? ia[t] : __ddiv_rn(1.0, Sa));
        ss.invSbf = invSbf;
        ss.invShf = __double2float_rn(ih ? ih[t] : __ddiv_rn(1.0, Sh));
        ss.LA = 0.6931472f * (1.0f + fmaxf(0.0f, -__log2f(__double2float_rn(Sa))));
        ss.keep = refresh_at(t, p.n_refresh) ? 0 : ~0;
        ss.ocol = row_at(p.order, t, p.T, p.grid) * p.E;
        const float qa1 = static_cast<float>((1 << (p.abits - 1)) - 1) + 1.0f;
        ss.hA1 = qa1 * ss.LA;
        ss.hA0 = 0.5f - fmaf(qa1, fmaf(ss.LA, 1.1920929e-7f, 4.7683716e-7f), 1e-6f);
        ss.pad[0] = ss.pad[1] = 0;
        ss.Saf = __double2float_rn(Sa);
        ss.Sbf = __double2float_rn(Sb);
        ss.Shf = __double2float_rn(Sh);
        ss.pad2 = 0.0f;
    }
    constexpr int kChunks16 = static_cast<int>(sizeof(StepShared) / 16);
    const uint4* src = reinterpret_cast<const uint4*>(&ss);
    const int s1 = min(S, s0 + kTabSamples);
    const size_t P2 = static_cast<size_t>(p.E) + 32;
    const double* col = p.proj + static_cast<size_t>(t) * P2 + p.E + lane;  // + s*T*P2 per sample
    double vs[kTabSamples];  // every sample's B / C row of this step, loaded at once
#pragma unroll
    for (int j = 0; j < kTabSamples; ++j)
        vs[j] = s0 + j < s1 ? col[static_cast<size_t>(s0 + j) * T * P2] : 0.0;
#pragma unroll
    for (int j = 0; j < kTabSamples; ++j) {
        const int s = s0 + j;
        if (s >= s1) break;
        const double v = vs[j];
        double bm = fabs(v);
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) bm = fmax(bm, __shfl_xor_sync(0xffffffffu, bm, o));
        float bs = 0.0f;
        __syncwarp();  // the previous sample's record has been copied out
        if (lane < 16) {
            bs = __double2float_rn(v) * invSbf;
            ss.B[lane] = v;
            ss.BSf[lane] = bs;
        } else {
            ss.C[lane - 16] = v;
        }
        bs = fabsf(bs);
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) bs = fmaxf(bs, __shfl_xor_sync(0xffffffffu, bs, o));
        if (lane == 0) {
            ss.Bmax = bm;
            ss.Bmaxf = __double2float_rn(bm);
            ss.BSmaxf = bs;
        }
        __syncwarp();
        uint4* dst = reinterpret_cast<uint4*>(out + (static_cast<size_t>(dd) * S + s) * T + t);
        for (int k = lane; k < kChunks16; k += 32) dst[k] = src[k];
    }
}

template <bool EXACT, int ABITS, bool TRACE, bool FS = false>
__global__ void __launch_bounds__(kThr, 8) k3_scan_fast(const ScanDirs P, const StepShared* __restrict__ steps) {
    extern __shared__ __align__(16) uint8_t scan_smem_raw[];
    const int warp = threadIdx.x >> 5;
    WarpSmem& sh = reinterpret_cast<WarpSmem*>(scan_smem_raw)[warp];
    const ScanParams& p = P.d[blockIdx.z];
    const unsigned lane = threadIdx.x & 31;
    const int s = blockIdx.y, c = lane >> 1, half = lane & 1;
    const int cw = blockIdx.x * kCh + warp * kWarpCh;  // first channel of this warp
    if (cw >= p.E) return;  // no CTA-wide barriers below
    const int i = cw + c;
    const bool active = i < p.E;
    const int E = p.E, T = p.T, P2 = E + 32, m0 = half * 8;
    const unsigned pair = 3u << (lane & ~1u);
    const bool dyn = p.mode == MODE_DYNAMIC;
    constexpr double qa = static_cast<double>((1 << (ABITS - 1)) - 1), qo = 127.0;  // outlier_bits = 8
    constexpr float qaf = static_cast<float>(qa), qof = 127.0f;
    const double* __restrict__ proj = p.proj;
    const double* __restrict__ uin = p.u;
    double* __restrict__ obase = p.o + static_cast<size_t>(s) * T * E + (active ? i : 0);
    const double* __restrict__ arow = p.a + static_cast<size_t>(active ? i : 0) * 16;
    float2 A2f[4];  // f32(A_m log2 e), pairs for the packed f32x2 pipe
    double Amax = -1e300;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double a0 = active ? arow[m0 + 2 * k] : -1.0, a1 = active ? arow[m0 + 2 * k + 1] : -1.0;
        A2f[k] = make_float2(__double2float_rn(a0 * 1.4426950408889634), __double2float_rn(a1 * 1.4426950408889634));
        Amax = fmax(Amax, fmax(a0, a1));
    }
    Amax = fmax(Amax, __shfl_xor_sync(0xffffffffu, Amax, 1));
    const float Amax2f = __double2float_rn(Amax * 1.4426950408889634);
    double h[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) h[m] = 0.0;
    unsigned fl = 0;  // channel in O: bit 0 a_bar, bit 1 b_bar, bit 2 h
    const double thA = p.cal[0].theta, thB = p.cal[1].theta, thH = p.cal[2].theta;
    const float thAf = __double2float_rn(thA), thBf = __double2float_rn(thB), thHf = __double2float_rn(thH);
    // FS (k3_scan_c1's f32 state update, 8 states per thread): previous h codes and scale
    float2 rhp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rhp[k] = make_float2(0.0f, 0.0f);
    float sHf_prev = 0.0f, qHp = 0.0f;
    double sHp = 0.0;
    const float thHlo = thHf * (1.0f - 4.0f * 5.9604645e-8f);
    // chunk staging: lane -> (step, channel) = (lane >> 4 + 2k, lane & 15)
    const int sc = lane & 15, sic = cw + sc;
    const double bd = sic < E ? p.b_delta[sic] : 0.0;
    const StepShared* wsteps = steps + (static_cast<size_t>(blockIdx.z) * p.S + s) * T;
    if (lane == 0) {
        ptx::mbar_init(&sh.bar[0], 1);
        ptx::mbar_init(&sh.bar[1], 1);
        ptx::fence_barrier_init();
    }
    __syncwarp();
    auto issue = [&](int t0, int buf) {  // async copies of chunk t0 into buffer buf
        const int nt = min(kChunk, T - t0);
#pragma unroll
        for (int k = 0; k < kChunk / 2; ++k) {
            const int tt = (lane >> 4) + 2 * k, t = min(t0 + tt, T - 1);
            const bool ok = tt < nt && sic < E;
            const int cr = row_at(p.order, t, T, p.grid);
            cp_async8(&sh.dp[buf][tt][sc], proj + (static_cast<size_t>(s) * T + t) * P2 + (ok ? sic : 0), ok);
            cp_async8(&sh.u[buf][tt][sc], uin + (static_cast<size_t>(s) * T + cr) * E + (ok ? sic : 0), ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (lane == 0) {
            const uint32_t bytes = static_cast<uint32_t>(nt * sizeof(StepShared));
            ptx::mbar_arrive_expect_tx(&sh.bar[buf], bytes);
            ptx::bulk_g2s(&sh.st[buf][0], wsteps + t0, bytes, &sh.bar[buf]);
        }
    };
    issue(0, 0);

    for (int t0 = 0, ci = 0; t0 < T; t0 += kChunk, ++ci) {
        const int nt = min(kChunk, T - t0), cur = ci & 1;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();  // chunk ci's per-channel inputs landed; chunk ci-1 consumed
#pragma unroll
        for (int k = 0; k < kChunk / 2; ++k) {
            const int tt = (lane >> 4) + 2 * k;
            const double x = dadd(sh.dp[cur][tt][sc], bd);  // softplus argument, ssm.cpp:150-151
            float eps;
            sh.x[tt][sc] = x;
            sh.deltaf[tt][sc] = softplus_f32(__double2float_rn(x), eps);
            sh.epsd[tt][sc] = eps;
        }
        if (t0 + kChunk < T) issue(t0 + kChunk, cur ^ 1);
        __syncwarp();
        ptx::mbar_wait(&sh.bar[cur], (ci >> 1) & 1);

        // Output of step tt (o = 0 + C_0 h_0 + ... + C_15 h_15 in order: the first lane of a
        // pair sums from 0, the second continues the same chain) from the carried state h,
        // which still holds step tt's quantized state until pass 2 of step tt+1 updates it.
        // For A4 it is issued from inside pass 1 of step tt+1, so its dependent DADD chain
        // overlaps that step's independent f32 work (measured 2.44 vs 2.49 ms per Vim-B
        // launch; A8 measured 3 % slower deferred, so it emits at the end of its step); the
        // chunk's last step is emitted at the end of the chunk (its step record is about to
        // be recycled).
        auto emit = [&](int te, unsigned fl_e, bool store) {
            const StepShared& se = sh.st[cur][te];
            double pr[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if constexpr (FS)  // the state is code * scale (fake_quant_step's dequantized value)
                    pr[m] = dmul(se.C[m0 + m], dmul(static_cast<double>((m & 1) ? rhp[m >> 1].y : rhp[m >> 1].x), sHp));
                else
                    pr[m] = dmul(se.C[m0 + m], h[m]);
            }
            double o = 0.0;
#pragma unroll
            for (int m = 0; m < 8; ++m) o = dadd(o, pr[m]);
            o = __shfl_sync(0xffffffffu, o, lane & ~1u);
#pragma unroll
            for (int m = 0; m < 8; ++m) o = dadd(o, pr[m]);
            if (store && half && active) {
                obase[se.ocol] = o;
                if constexpr (TRACE) {
                    const size_t b = (static_cast<size_t>(s) * T + t0 + te) * E + i;
                    const size_t kst = static_cast<size_t>(p.S) * T * E;
                    p.masks[b] = fl_e & 1u;
                    p.masks[kst + b] = (fl_e >> 1) & 1u;
                    p.masks[2 * kst + b] = (fl_e >> 2) & 1u;
                }
            }
        };
        constexpr bool kDefer = ABITS == 4;
        unsigned fl_prev = fl;
        for (int tt = 0; tt < nt; ++tt) {
            const StepShared& ss = sh.st[cur][tt];
            const float df = sh.deltaf[tt][c];
            const float ed = sh.epsd[tt][c];
            const double uv = sh.u[cur][tt][c];
            // exact delta and peaks, computed on demand (decisions near theta, outlier
            // scales, fallbacks)
            bool have = false;
            double delta, pa, pb;
            auto exact = [&]() {
                if (!have) {
                    delta = softplus_call(sh.x[tt][c]);
                    pa = exp_call(dmul(delta, Amax));
                    pb = dmul(delta, ss.Bmax);
                    have = true;
                }
            };
            // inlier scales (static mode; dynamic steps where neither tensor is an outlier)
            double sA = ss.Sa, sB = ss.Sb;
            float invA = ss.invSaf, kB = 1.0f, qAf = qaf, qBf = qaf;
            // Certification margins (in units of q) where rounding matters (|q| <= qmax+1):
            // a_bar: |dq| <= q (ln2 |x2| (ed + 2^-23) + 2^-21), ln2 |x2| <= LA there;
            // b_bar: |dq| <= |q| (ed + 8 2^-24). Inlier forms folded to h0 - h1*ed.
            float halfA = fmaf(-ss.hA1, ed, ss.hA0);
            float halfB = fmaf(-(qaf + 1.0f), ed, 0.5f - fmaf(qaf + 1.0f, 4.7683716e-7f, 1e-6f));
            // f32 a_bar peak: the detector's certified estimate and the clipping bound below
            const float x2m = df * Amax2f;
            const float paf = ex2_approx(x2m);
            if (dyn) {
                fl &= static_cast<unsigned>(ss.keep);  // maybe_refresh, quant.cpp:303-311
                // detect_outliers, channel-local form, on certified f32 peaks
                const float ea = 2.0f * fmaf(0.6931472f * fabsf(x2m), ed + 1.1920929e-7f, 4.7683716e-7f) + 1e-6f;
                const float pbf = df * ss.Bmaxf;
                const float eb = 2.0f * (ed + 2.3841858e-7f) + 1e-6f;
                // one branch off the inlier path: outlier channels and decisions within the bound
                if ((fl & 3u) | (paf >= thAf * (1.0f - ea)) | (pbf >= thBf * (1.0f - eb))) {
                    if (!(fl & 1u)) {
                        if (paf > thAf * (1.0f + ea)) {
                            fl |= 1u;
                        } else if (paf >= thAf * (1.0f - ea)) {
                            exact();
                            if (pa > thA) fl |= 1u;
                        }
                    }
                    if (!(fl & 2u)) {
                        if (pbf > thBf * (1.0f + eb)) {
                            fl |= 2u;
                        } else if (pbf >= thBf * (1.0f - eb)) {
                            exact();
                            if (pb > thB) fl |= 2u;
                        }
                    }
                    if (fl & 3u) exact();
                    if (fl & 1u) {
                        sA = scale_call(pa, qo);
                        invA = __double2float_rn(recip_call(sA));
                        qAf = qof;
                        const float LA = 0.6931472f * (1.0f + fmaxf(0.0f, -__log2f(__double2float_rn(sA))));
                        halfA = 0.5f - fmaf(qAf + 1.0f, fmaf(LA, ed + 1.1920929e-7f, 4.7683716e-7f), 1e-6f);
                    }
                    if (fl & 2u) {
                        sB = scale_call(pb, qo);
                        kB = __double2float_rn(recip_call(sB)) / ss.invSbf;
                        qBf = qof;
                        halfB = 0.5f - fmaf(qBf + 1.0f, ed + 4.7683716e-7f, 1e-6f);
                    }
                }
            }
            const float dfb = df * kB;
            const float capA = qAf + 0.25f, capB = qBf + 0.25f;
            // pass 1: codes from the f32 quotients (round-to-nearest via 1.5*2^23), clamped
            // before rounding so the integer is the reference's clipped code. Two elements
            // per packed f32x2 instruction; codes are kept as magic bit patterns.
            unsigned ca[8];  // a_bar codes (>= 0) as integers, b_bar codes as exact f32 integers
            float cb[8];
            float raf[8];  // FS: a_bar codes as exact f32 integers
            bool redo = EXACT || sA < 1e-30;  // ex2.approx.ftz flushes below 2^-126
            const float2* BS2 = reinterpret_cast<const float2*>(ss.BSf + m0);
            auto pass1 = [&](auto clamp) {
                constexpr bool CL = decltype(clamp)::value;
                if constexpr (kDefer)
                    if (tt > 0) emit(tt - 1, fl_prev, true);  // previous step's output (see emit)
                float mda = 0.0f, mdb = 0.0f;  // largest distance to the rounded code (3-input max)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float2 x2 = __fmul2_rn(f2(df), A2f[k]);
                    float2 qa2 = __fmul2_rn(make_float2(ex2_approx(x2.x), ex2_approx(x2.y)), f2(invA));
                    if constexpr (CL) {
                        qa2.x = fminf(qa2.x, capA);
                        qa2.y = fminf(qa2.y, capA);
                    }
                    const float2 ta = __fadd2_rn(qa2, f2(12582912.0f));
                    const float2 ra = __fadd2_rn(ta, f2(-12582912.0f));
                    const float2 da = __fadd2_rn(qa2, make_float2(-ra.x, -ra.y));
                    if constexpr (FS) {
                        raf[2 * k] = ra.x;
                        raf[2 * k + 1] = ra.y;
                    } else {
                        ca[2 * k] = __float_as_uint(ta.x) - kMagicBits;
                        ca[2 * k + 1] = __float_as_uint(ta.y) - kMagicBits;
                    }
                    float2 qb2 = __fmul2_rn(f2(dfb), BS2[k]);
                    if constexpr (CL) {
                        qb2.x = fminf(fmaxf(qb2.x, -capB), capB);
                        qb2.y = fminf(fmaxf(qb2.y, -capB), capB);
                    }
                    const float2 tb = __fadd2_rn(qb2, f2(12582912.0f));
                    const float2 rb = __fadd2_rn(tb, f2(-12582912.0f));
                    const float2 db = __fadd2_rn(qb2, make_float2(-rb.x, -rb.y));
                    cb[2 * k] = rb.x;
                    cb[2 * k + 1] = rb.y;
                    mda = fmaxf(mda, fmaxf(fabsf(da.x), fabsf(da.y)));
                    mdb = fmaxf(mdb, fmaxf(fabsf(db.x), fabsf(db.y)));
                }
                redo |= (mda > halfA) | (mdb > halfB);
            };
            // The clamps can bind only if the largest quotient exceeds the cap: q_b <=
            // dfb*max|BSf| and q_a <= paf*invA (monotone rounding; the factor covers
            // ex2.approx's relative error). Warp-uniform choice, both forms are exact.
            const bool noclip = dfb * ss.BSmaxf <= capB && paf * invA * 1.000001f <= capA;
            if (__all_sync(0xffffffffu, noclip)) pass1(std::false_type{});
            else pass1(std::true_type{});
            if (redo) {  // exact f64 codes where the f32 quotient is not certified
                exact();
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const float a2 = (m & 1) ? A2f[m >> 1].y : A2f[m >> 1].x;
                    const float qa_f = fminf(ex2_approx(df * a2) * invA, capA);
                    if (EXACT || sA < 1e-30 || fabsf(qa_f - rintf(qa_f)) > halfA) {
                        const double cq = qdiv_call(exp_call(dmul(delta, arow[m0 + m])), sA, static_cast<double>(qAf));
                        ca[m] = static_cast<unsigned>(static_cast<int>(cq));
                        raf[m] = static_cast<float>(cq);
                    }
                    const float qb_f = fminf(fmaxf(dfb * ss.BSf[m0 + m], -capB), capB);
                    if (EXACT || fabsf(qb_f - rintf(qb_f)) > halfB)
                        cb[m] = static_cast<float>(
                            qdiv_call(dmul(delta, ss.B[m0 + m]), sB, static_cast<double>(qBf)));
                }
            }
            if constexpr (FS) {
                // f32 state update with its bound (k3_scan_c1<FS>'s header comment), 8 states per
                // thread; the pair shares the channel's peak, detector decision and exact path
                const float sAf = (fl & 1u) ? __double2float_rn(sA) : ss.Saf;
                const float sBf = (fl & 2u) ? __double2float_rn(sB) : ss.Sbf;
                const float sAsH = sAf * sHf_prev, sBu = sBf * __double2float_rn(uv);
                float2 hf2[4];
                float phf = 0.0f;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float2 p1 = __fmul2_rn(__fmul2_rn(make_float2(raf[2 * k], raf[2 * k + 1]), rhp[k]), f2(sAsH));
                    const float2 p2 = __fmul2_rn(make_float2(cb[2 * k], cb[2 * k + 1]), f2(sBu));
                    const float2 hv = __fadd2_rn(p1, p2);
                    phf = fmaxf(phf, fmaxf(fabsf(hv.x), fabsf(hv.y)));
                    hf2[k] = hv;
                }
                phf = fmaxf(phf, __shfl_xor_sync(0xffffffffu, phf, 1));
                const float maxD = fmaf(fmaf(qAf * qHp, sAsH, qBf * fabsf(sBu)), 5.3f * 5.9604645e-8f, 1e-37f);
                double sH = ss.Sh, qH = qa;
                float invHf = ss.invShf;
                bool hexact = EXACT || !(maxD < 1e30f);
                if (dyn) hexact |= (fl & 4u) || !(fmaf(maxD, 1.0000003f, phf) < thHlo);
                const float capH = qaf + 0.25f;
                const float halfH = 0.5f - fmaf(maxD, invHf * 1.0001f, fmaf(qaf + 1.0f, 1.25e-7f, 1e-6f));
                float chd[8];
                float mdh = 0.0f;
                auto hcodes = [&](auto clamp) {
                    constexpr bool CL = decltype(clamp)::value;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        float2 q = __fmul2_rn(hf2[k], f2(invHf));
                        if constexpr (CL) {
                            q.x = fminf(fmaxf(q.x, -capH), capH);
                            q.y = fminf(fmaxf(q.y, -capH), capH);
                        }
                        const float2 th = __fadd2_rn(q, f2(12582912.0f));
                        const float2 rh = __fadd2_rn(th, f2(-12582912.0f));
                        const float2 dh = __fadd2_rn(q, make_float2(-rh.x, -rh.y));
                        chd[2 * k] = rh.x;
                        chd[2 * k + 1] = rh.y;
                        mdh = fmaxf(mdh, fmaxf(fabsf(dh.x), fabsf(dh.y)));
                    }
                };
                if (__all_sync(0xffffffffu, phf * invHf <= capH)) hcodes(std::false_type{});
                else hcodes(std::true_type{});
                hexact |= !(mdh <= halfH);
                hexact |= __shfl_xor_sync(0xffffffffu, hexact ? 1 : 0, 1) != 0;  // the pair decides together
                if (hexact) {  // the exact f64 update (ssm.cpp:165-167) and the f64-state h logic on it
                    double hn[8];
#pragma unroll
                    for (int m = 0; m < 8; ++m) {
                        const double a_q = dmul(static_cast<double>(raf[m]), sA);
                        const double b_q = dmul(static_cast<double>(cb[m]), sB);
                        const double hp = dmul(static_cast<double>((m & 1) ? rhp[m >> 1].y : rhp[m >> 1].x), sHp);
                        hn[m] = dadd(dmul(a_q, hp), dmul(b_q, uv));
                    }
                    if (dyn) {
                        double ph = 0.0;
#pragma unroll
                        for (int m = 0; m < 8; ++m) ph = fmax(ph, fabs(hn[m]));
                        ph = fmax(ph, __shfl_xor_sync(pair, ph, 1));
                        if (ph > thH) fl |= 4u;
                        if (fl & 4u) {
                            sH = scale_call(ph, qo);
                            invHf = __double2float_rn(recip_call(sH));
                            qH = qo;
                        }
                    }
                    const float qHf = static_cast<float>(qH), capHx = qHf + 0.25f;
                    const float halfHx = 0.5f - fmaf(qHf + 1.0f, 2.3841858e-7f, 1e-6f);
#pragma unroll
                    for (int m = 0; m < 8; ++m) {  // |dq| <= |q| 4 2^-24 from the exact value
                        const float q = fminf(fmaxf(__double2float_rn(hn[m]) * invHf, -capHx), capHx);
                        const float r = rintf(q);
                        chd[m] = (EXACT || !(fabsf(q - r) <= halfHx)) ? static_cast<float>(qdiv_call(hn[m], sH, qH)) : r;
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) rhp[k] = make_float2(chd[2 * k], chd[2 * k + 1]);  // carried state
                sHp = sH;
                sHf_prev = (fl & 4u) ? __double2float_rn(sH) : ss.Shf;
                qHp = static_cast<float>(qH);
            } else {
            // pass 2: dequantized values (code * s, fake_quant_step) and the exact f64 update.
                // a_bar codes are >= 0: fma(2^52 + c, sA, -2^52 sA) = c sA before its one rounding,
                // i.e. exactly dmul(c, sA).
                const double nKA = dmul(sA, -4503599627370496.0);
    #pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const double a_q = __fma_rn(__hiloint2double(0x43300000, static_cast<int>(ca[m])), sA, nKA);
                    const double b_q = dmul(static_cast<double>(cb[m]), sB);
                    h[m] = dadd(dmul(a_q, h[m]), dmul(b_q, uv));  // ssm.cpp:165-167
                }
                // h detection + codes. Rounding to f32 is monotone, so the f32 peak
                // max_m fl32|h_m| equals fl32(max_m |h_m|): phf > fl32(theta) implies
                // peak > theta, phf < fl32(theta) implies peak <= theta; only equality
                // needs the exact f64 peak. Outlier channels take the exact peak for their scale.
                float2 hfv[4];
                float phf = 0.0f;
    #pragma unroll
                for (int k = 0; k < 4; ++k) {
                    hfv[k] = make_float2(__double2float_rn(h[2 * k]), __double2float_rn(h[2 * k + 1]));
                    phf = fmaxf(phf, fmaxf(fabsf(hfv[k].x), fabsf(hfv[k].y)));
                }
                phf = fmaxf(phf, __shfl_xor_sync(0xffffffffu, phf, 1));
                double sH = ss.Sh, qH = qa;
                float invHf = ss.invShf;
                if (dyn && ((fl & 4u) | (phf >= thHf))) {
                    if (!(fl & 4u)) {
                        if (phf > thHf) {
                            fl |= 4u;
                        } else {  // phf == fl32(theta): the exact peak decides
                            double ph = 0.0;
    #pragma unroll
                            for (int m = 0; m < 8; ++m) ph = fmax(ph, fabs(h[m]));
                            ph = fmax(ph, __shfl_xor_sync(pair, ph, 1));
                            if (ph > thH) fl |= 4u;
                        }
                    }
                    if (fl & 4u) {
                        double ph = 0.0;
    #pragma unroll
                        for (int m = 0; m < 8; ++m) ph = fmax(ph, fabs(h[m]));
                        ph = fmax(ph, __shfl_xor_sync(pair, ph, 1));
                        sH = scale_call(ph, qo);
                        invHf = __double2float_rn(recip_call(sH));
                        qH = qo;
                    }
                }
                {  // |dq| <= |q| 4 2^-24 (h and 1/s rounded to f32, one product)
                    const float qHf = static_cast<float>(qH), capH = qHf + 0.25f;
                    const float halfH = 0.5f - fmaf(qHf + 1.0f, 2.3841858e-7f, 1e-6f);
                    float chd[8];  // h codes as exact f32 integers (F2F.F64 balances the XU and FP64 pipes)
                    bool hredo = EXACT;
                    auto hcodes = [&](auto clamp) {
                        constexpr bool CL = decltype(clamp)::value;
                        float mdh = 0.0f;
    #pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            float2 q = __fmul2_rn(hfv[k], f2(invHf));
                            if constexpr (CL) {
                                q.x = fminf(fmaxf(q.x, -capH), capH);
                                q.y = fminf(fmaxf(q.y, -capH), capH);
                            }
                            const float2 th = __fadd2_rn(q, f2(12582912.0f));
                            const float2 rh = __fadd2_rn(th, f2(-12582912.0f));
                            const float2 dh = __fadd2_rn(q, make_float2(-rh.x, -rh.y));
                            chd[2 * k] = rh.x;
                            chd[2 * k + 1] = rh.y;
                            mdh = fmaxf(mdh, fmaxf(fabsf(dh.x), fabsf(dh.y)));
                        }
                        hredo |= mdh > halfH;
                    };
                    if (__all_sync(0xffffffffu, phf * invHf <= capH)) hcodes(std::false_type{});  // |q| <= phf*invHf
                    else hcodes(std::true_type{});
                    if (hredo) {
    #pragma unroll
                        for (int m = 0; m < 8; ++m) {
                            const float hv = (m & 1) ? hfv[m >> 1].y : hfv[m >> 1].x;
                            const float q = fminf(fmaxf(hv * invHf, -capH), capH);
                            if (EXACT || fabsf(q - rintf(q)) > halfH)
                                chd[m] = static_cast<float>(qdiv_call(h[m], sH, qH));
                        }
                    }
    #pragma unroll
                    for (int m = 0; m < 8; ++m) h[m] = dmul(static_cast<double>(chd[m]), sH);  // carried state
                }
            }
            if constexpr (!kDefer) emit(tt, fl, true);
            fl_prev = fl;
        }
        if constexpr (kDefer) emit(nt - 1, fl_prev, true);
    }
}

// ---- the out_proj input K1 fused into the scan ----------------
// k1_channel's merge source (k1_detect_quant.cu) for one (sample, 32-channel group)
// with lane = channel walking the T tokens in canonical order: merged = (0 + o_0) +
// o_1 (ssm.cpp:214-229), v = merged * silu(gate) certified in f32 (merge_f32.cuh),
// maybe_refresh / detect_outliers in the channel-local form, split_quantize's codes;
// the group's 32 channels are one mask word (a ballot) and |O(t)| is accumulated
// across the E/32 groups with one atomic per row. The scan outputs o_d come from L2
// (the other direction's CTA of the same group ran alongside: dir is the grid's
// fastest index); the next tokens' operands are in flight while one is quantized.
__device__ __noinline__ double merge_exact_call(double m, double g) { return dmul(m, silu_d(g)); }

__device__ void merge_tail(const K1Params& p, int s, int grp, unsigned lane) {
    const int E = p.E, T = p.T, J = E >> 5, i = grp * 32 + static_cast<int>(lane);
    const bool dyn = p.mode == MODE_DYNAMIC;
    const double qa = qmax_for(p.abits), qo = qmax_for(p.obits);
    const int qai = static_cast<int>(qa);
    const double theta = p.cal.theta;
    const float thetaf = __double2float_rn(theta), capf = static_cast<float>(qa) + 1.0f;
    const double* __restrict__ s_tab = dyn ? p.cal.s_in : p.cal.s_full;
    const double* __restrict__ i_tab = dyn ? p.inv_in : p.inv_full;
    const size_t base = static_cast<size_t>(s) * T;
    constexpr int kG = 4;  // tokens per group; the next group's loads are issued before this one is used
    double o0[2][kG], o1[2][kG], gt[2][kG];
    auto load = [&](int b, int t0) {
#pragma unroll
        for (int k = 0; k < kG; ++k) {
            const int t = min(t0 + k, T - 1);
            const size_t idx = (base + t) * E + i;
            o0[b][k] = __ldcg(p.x + idx);
            o1[b][k] = p.x2 ? __ldcg(p.x2 + idx) : 0.0;
            gt[b][k] = __ldg(p.gate + idx);
        }
    };
    load(0, 0);
    bool in = false;
    for (int t0 = 0, b = 0; t0 < T; t0 += kG, b ^= 1) {
        if (t0 + kG < T) {
            if (b) load(0, t0 + kG);
            else load(1, t0 + kG);
        }
#pragma unroll
        for (int k = 0; k < kG; ++k) {
            const int t = t0 + k;
            if (t >= T) break;
            const size_t row = base + t;
            const double a0 = b ? o0[1][k] : o0[0][k], a1 = b ? o1[1][k] : o1[0][k];
            const double g = b ? gt[1][k] : gt[0][k];
            double mg = dadd(0.0, a0);  // (0 + o_0) + o_1
            if (p.x2) mg = dadd(mg, a1);
            const MergeApprox ap = merge_approx(mg, g);
            bool have = false;
            double v = 0.0;
            if (dyn) {
                if (refresh_at(t, p.n_refresh)) in = false;  // maybe_refresh
                if (!in) {                                   // detect_outliers, channel-local form
                    const float av = fabsf(ap.v);
                    if (av * (1.0f - ap.eps) > thetaf * 1.0000003f) {
                        in = true;
                    } else if (av * (1.0f + ap.eps) >= thetaf * 0.9999997f) {
                        v = merge_exact_call(mg, g);
                        have = true;
                        in = fabs(v) > theta;
                    }
                }
            }
            const double S = s_tab[t];
            const double inv = i_tab ? i_tab[t] : __ddiv_rn(1.0, S);
            int c = 0;
            if (in) {
                if (!have) v = merge_exact_call(mg, g);
                const double os = scale_from_peak(fabs(v), qo);  // scale_for over the 1-value row
                p.ocode[row * E + i] = static_cast<int8_t>(static_cast<int>(quant_code_div(v, os, qo)));
                p.oscale[row * E + i] = os;
            } else {
                // certified f32 quotient: |dq| <= (|q| + 1) (eps + 3 2^-24)
                const float q = fminf(fmaxf(ap.v * __double2float_rn(inv), -capf), capf);
                const float r = rintf(q);
                if (!have && fabsf(q - r) < 0.5f - fmaf(fabsf(q) + 1.0f, ap.eps + 1.8e-7f, 1e-6f)) {
                    c = min(max(static_cast<int>(r), -qai), qai);
                } else {
                    if (!have) v = merge_exact_call(mg, g);
                    c = quant_code_int(v, S, inv, qa, qai);
                }
            }
            if (p.codes4) {  // lanes 2j, 2j+1: one pack_int4 byte
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

// ---- one thread per channel ---------------------------------------------------
// Same arithmetic as k3_scan_fast (every certification bound above holds
// unchanged), with lane = channel and all N = 16 states in one thread: the
// per-step work that does not scale with the states (step-record loads,
// detection, votes, branches, the output store) is paid once per 32 channels
// instead of once per 16, and the output sum 0 + C_0 h_0 + ... + C_15 h_15 is
// one in-order chain in one thread (no half-duplicated additions, no shuffles).
// A chunk pre-pass evaluates, per (step, channel) with the chunk's steps as
// independent streams, the f32 delta, the inlier certification margins, the
// detector's "near or above theta" flag and the clamp flag; the step loop reads
// them with one 16-byte shared load.
//
// FS (f32 state update). The carried state is h' = rh' * S_h' (codes rh', exact f32
// integers, and the previous step's scale), so no f64 state is kept. The update
// h = fl64(fl64(a_q h') + fl64(b_q u)) (ssm.cpp:165-167) is evaluated in f32 as
//   P1 = fl32(fl32(ra * rh') * fl32(f32(S_a) f32(S_h'))),  P2 = fl32(rb * fl32(f32(S_b) f32(u))),
//   hf = fl32(P1 + P2)
// (ra, rb: the a_bar / b_bar codes; ra * rh' <= 127^2 is exact). Each of P1, P2 is
// within 4.0002 u of its f64 counterpart (u = 2^-24: four / three roundings of
// exact inputs, against 2^-53 ones), the sum and the f64 roundings add u |P1 + P2|
// and 2^-53 (|A| + |B|), so |hf - h| <= (|P1| + |P2|) 5.01 u <= D = (max|P1| +
// max|P2|) 5.2 u + 1e-37 (the absolute term covers f32 underflow). Then:
//  * code: q = fl32(hf * invH) is within |q| 2.001 u + D invH 1.0001 of h / S_h, so
//    round(q) is the reference's code when |q - round(q)| <= 0.5 - that (clamped
//    quotients as in the f64-state form);
//  * detector (dynamic): max|h| < theta is certain when max|hf| + D < theta (rounded
//    down); h-outlier channels, peaks not certainly below theta, non-finite values
//    and uncertified codes take the exact path: the f64 update from the codes and
//    scales, then the f64-state form's detection and codes.
// The output o = sum C_m (rh_m * S_h) is the reference's f64 sum of the dequantized
// state.
template <int KC>
struct C1Smem {
    StepShared st[2][KC];
    double dp[2][KC][32];  // x_proj delta pre-activations (raw), lane = channel
    double u[2][KC][32];
    float4 pre[KC][32];    // df, inlier halfA, inlier halfB, flags (bit 0 detect, bit 1 clamp)
    float4 a2[4][32];      // SMA2: f32(A_m log2 e) of the lane's channel (frees 16 registers)
    uint64_t bar[2];
};

template <bool EXACT, int ABITS, bool TRACE, int KC, int MINB, bool FS, bool SMA2 = false, bool MT = false>
__global__ void __launch_bounds__(32, MINB) k3_scan_c1(const ScanDirs P, const StepShared* __restrict__ steps) {
    extern __shared__ __align__(16) uint8_t c1_smem_raw[];
    using Sm = C1Smem<KC>;
    Sm& sh = *reinterpret_cast<Sm*>(c1_smem_raw);
    // grid x = channel group * n + direction: the directions of a (sample, group) run side by
    // side (the fused merge tail reads both outputs from L2)
    const int dir = P.n == 2 ? static_cast<int>(blockIdx.x & 1) : 0;
    const int grp = P.n == 2 ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const ScanParams& p = P.d[dir];
    const unsigned lane = threadIdx.x & 31;
    const int s = blockIdx.y;
    const int cw = grp * 32;  // first channel of this warp (CTA = one warp)
    const int i = cw + static_cast<int>(lane);
    const bool active = i < p.E;
    const int E = p.E, T = p.T, P2 = E + 32;
    const bool dyn = p.mode == MODE_DYNAMIC;
    constexpr double qa = static_cast<double>((1 << (ABITS - 1)) - 1), qo = 127.0;  // outlier_bits = 8
    constexpr float qaf = static_cast<float>(qa), qof = 127.0f;
    const double* __restrict__ proj = p.proj;
    const double* __restrict__ uin = p.u;
    double* __restrict__ obase = p.o + static_cast<size_t>(s) * T * E + (active ? i : 0);
    const double* __restrict__ arow = p.a + static_cast<size_t>(active ? i : 0) * 16;
    float2 A2r[SMA2 ? 1 : 8];  // f32(A_m log2 e), pairs for the packed f32x2 pipe (registers or shared)
    double Amax = -1e300;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const double a0 = active ? arow[2 * k] : -1.0, a1 = active ? arow[2 * k + 1] : -1.0;
        const float2 v = make_float2(__double2float_rn(a0 * 1.4426950408889634), __double2float_rn(a1 * 1.4426950408889634));
        if constexpr (SMA2) reinterpret_cast<float2*>(&sh.a2[k >> 1][lane])[k & 1] = v;
        else A2r[k] = v;
        Amax = fmax(Amax, fmax(a0, a1));
    }
    auto A2f_at = [&](int k) -> float2 {
        if constexpr (SMA2) return reinterpret_cast<const float2*>(&sh.a2[k >> 1][lane])[k & 1];
        else return A2r[k];
    };
    const float Amax2f = __double2float_rn(Amax * 1.4426950408889634);
    double h[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) h[m] = 0.0;
    unsigned fl = 0;  // channel in O: bit 0 a_bar, bit 1 b_bar, bit 2 h
    const double thA = p.cal[0].theta, thB = p.cal[1].theta, thH = p.cal[2].theta;
    const float thAf = __double2float_rn(thA), thBf = __double2float_rn(thB), thHf = __double2float_rn(thH);
    // FS: the previous step's h codes (exact f32 integers) and f32 h scale; thHlo <= theta
    float2 rhp[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) rhp[k] = make_float2(0.0f, 0.0f);
    float sHf_prev = 0.0f, qHp = 0.0f;  // FS: f32 of the previous step's h scale, its code bound
    double sHp = 0.0;  // FS: the previous step's h scale; the state is rhp * sHp, exact (no f64 state kept)
    const float thHlo = thHf * (1.0f - 4.0f * 5.9604645e-8f);
    const double bd = active ? p.b_delta[i] : 0.0;
    const StepShared* wsteps = steps + (static_cast<size_t>(dir) * p.S + s) * T;
    if (lane == 0) {
        ptx::mbar_init(&sh.bar[0], 1);
        ptx::mbar_init(&sh.bar[1], 1);
        ptx::fence_barrier_init();
    }
    __syncwarp();
    const uint32_t rowbytes = static_cast<uint32_t>(min(32, E - cw)) * 8u;  // E even: a multiple of 16
    // chunk t0 into buffer buf: lane tt < nt bulk-copies step t0 + tt's x_proj delta row
    // and its scan input row (canonical position) for the warp's 32 channels; lane 0 the
    // step records; all complete on the buffer's mbarrier
    auto issue = [&](int t0, int buf) {
        const int nt = min(KC, T - t0);
        if (lane == 0)
            ptx::mbar_arrive_expect_tx(&sh.bar[buf], static_cast<uint32_t>(nt) * (sizeof(StepShared) + 2u * rowbytes));
        __syncwarp();
        if (static_cast<int>(lane) < nt) {
            const int t = t0 + static_cast<int>(lane);
            const int cr = row_at(p.order, t, T, p.grid);
            ptx::bulk_g2s(&sh.dp[buf][lane][0], proj + (static_cast<size_t>(s) * T + t) * P2 + cw, rowbytes, &sh.bar[buf]);
            ptx::bulk_g2s(&sh.u[buf][lane][0], uin + (static_cast<size_t>(s) * T + cr) * E + cw, rowbytes, &sh.bar[buf]);
        }
        if (lane == 0) ptx::bulk_g2s(&sh.st[buf][0], wsteps + t0, static_cast<uint32_t>(nt * sizeof(StepShared)), &sh.bar[buf]);
    };
    issue(0, 0);
    constexpr bool kDefer = ABITS == 4;
    const float hBc = 0.5f - fmaf(qaf + 1.0f, 4.7683716e-7f, 1e-6f);

    for (int t0 = 0, ci = 0; t0 < T; t0 += KC, ++ci) {
        const int nt = min(KC, T - t0), cur = ci & 1;
        __syncwarp();  // chunk ci-1 consumed
        ptx::mbar_wait(&sh.bar[cur], (ci >> 1) & 1);
        // pre-pass: per step of the chunk, this channel's f32 delta (softplus with its
        // bound), the certified a_bar peak, the detector flag and the inlier margins
#pragma unroll
        for (int tt = 0; tt < KC; ++tt) {
            const StepShared& ss = sh.st[cur][tt];
            const double x = dadd(sh.dp[cur][tt][lane], bd);  // softplus argument, ssm.cpp:150-151
            float ed;
            const float df = softplus_f32(__double2float_rn(x), ed);
            const float x2m = df * Amax2f;
            const float paf = ex2_approx(x2m);
            const float ea = 2.0f * fmaf(0.6931472f * fabsf(x2m), ed + 1.1920929e-7f, 4.7683716e-7f) + 1e-6f;
            const float pbf = df * ss.Bmaxf;
            const float eb = 2.0f * (ed + 2.3841858e-7f) + 1e-6f;
            const bool det = (paf >= thAf * (1.0f - ea)) | (pbf >= thBf * (1.0f - eb));
            const bool clip = !(df * ss.BSmaxf <= qaf + 0.25f && paf * ss.invSaf * 1.000001f <= qaf + 0.25f);
            sh.pre[tt][lane] = make_float4(df, fmaf(-ss.hA1, ed, ss.hA0), fmaf(-(qaf + 1.0f), ed, hBc),
                                           __uint_as_float((det ? 1u : 0u) | (clip ? 2u : 0u)));
        }
        if (t0 + KC < T) issue(t0 + KC, cur ^ 1);

        // output of step te from the carried state (see k3_scan_fast's emit); A4 issues it
        // from inside pass 1 of step te+1 so its DADD chain overlaps independent f32 work
        auto emit = [&](int te, unsigned fl_e) {
            const StepShared& se = sh.st[cur][te];
            const double2* C2 = reinterpret_cast<const double2*>(se.C);
            double o = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double2 c = C2[k];
                if constexpr (FS) {  // h = code * s (fake_quant_step's dequantized state), then C h
                    o = dadd(o, dmul(c.x, dmul(static_cast<double>(rhp[k].x), sHp)));
                    o = dadd(o, dmul(c.y, dmul(static_cast<double>(rhp[k].y), sHp)));
                } else {
                    o = dadd(o, dmul(c.x, h[2 * k]));
                    o = dadd(o, dmul(c.y, h[2 * k + 1]));
                }
            }
            if (active) {
                obase[se.ocol] = o;
                if constexpr (TRACE) {
                    const size_t b = (static_cast<size_t>(s) * T + t0 + te) * E + i;
                    const size_t kst = static_cast<size_t>(p.S) * T * E;
                    p.masks[b] = fl_e & 1u;
                    p.masks[kst + b] = (fl_e >> 1) & 1u;
                    p.masks[2 * kst + b] = (fl_e >> 2) & 1u;
                }
            }
        };
        unsigned fl_prev = fl;
#pragma unroll 1
        for (int tt = 0; tt < nt; ++tt) {
            const StepShared& ss = sh.st[cur][tt];
            const float4 pr = sh.pre[tt][lane];
            const float df = pr.x;
            const unsigned pf = __float_as_uint(pr.w);
            const double uv = sh.u[cur][tt][lane];
            bool have = false;
            double delta, pa, pb;
            auto exact = [&]() {
                if (!have) {
                    delta = softplus_call(dadd(sh.dp[cur][tt][lane], bd));
                    pa = exp_call(dmul(delta, Amax));
                    pb = dmul(delta, ss.Bmax);
                    have = true;
                }
            };
            double sA = ss.Sa, sB = ss.Sb;
            float invA = ss.invSaf, kB = 1.0f, qAf = qaf, qBf = qaf;
            float halfA = pr.y, halfB = pr.z;
            bool clip = pf & 2u;
            // FS: an outlier channel's scale (scale_for of its row, quant.cpp:37-42) as a
            // certified f32 estimate sXf with relative error epsX; the exact f64 scale is
            // computed only where an exact value is needed (sXexact false until then)
            float sAfo = 0.0f, sBfo = 0.0f, epsA = 0.0f, epsB = 0.0f;
            bool sAexact = true, sBexact = true;
            auto exact_scales = [&]() {
                if (!sAexact || !sBexact) exact();
                if (!sAexact) sA = scale_call(pa, qo);
                if (!sBexact) sB = scale_call(pb, qo);
                sAexact = sBexact = true;
            };
            if (dyn) {
                fl &= static_cast<unsigned>(ss.keep);  // maybe_refresh, quant.cpp:303-311
                // detect_outliers, channel-local form: only outlier channels and certified-peak
                // decisions within the bound of theta leave the inlier path
                if ((fl & 3u) | (pf & 1u)) {
                    float ed;
                    softplus_f32(__double2float_rn(dadd(sh.dp[cur][tt][lane], bd)), ed);
                    const float x2m = df * Amax2f;
                    const float paf = ex2_approx(x2m);
                    const float ea = 2.0f * fmaf(0.6931472f * fabsf(x2m), ed + 1.1920929e-7f, 4.7683716e-7f) + 1e-6f;
                    const float pbf = df * ss.Bmaxf;
                    const float eb = 2.0f * (ed + 2.3841858e-7f) + 1e-6f;
                    if (!(fl & 1u)) {
                        if (paf > thAf * (1.0f + ea)) {
                            fl |= 1u;
                        } else if (paf >= thAf * (1.0f - ea)) {
                            exact();
                            if (pa > thA) fl |= 1u;
                        }
                    }
                    if (!(fl & 2u)) {
                        if (pbf > thBf * (1.0f + eb)) {
                            fl |= 2u;
                        } else if (pbf >= thBf * (1.0f - eb)) {
                            exact();
                            if (pb > thB) fl |= 2u;
                        }
                    }
                    if (fl & 3u) {
                        if constexpr (FS) {
                            // sA = max a_bar / 127 = paf / 127 within eta_a (paf's bound) + 2.2 u; sB =
                            // delta max|B| / 127 = pbf / 127 within ed + 5.2 u. The quotient margins
                            // grow by these; codes stay certified against the exact scales
                            if (fl & 1u) {
                                epsA = fmaf(0.6931472f * fabsf(x2m), ed + 1.1920929e-7f, 4.7683716e-7f) + 1.32e-7f;
                                sAfo = paf * (1.0f / 127.0f);
                                sAexact = false;
                                invA = __frcp_rn(sAfo);
                                qAf = qof;
                                const float LA = 0.6931472f * (1.001f + fmaxf(0.0f, -__log2f(sAfo)));
                                halfA = 0.5f - fmaf(qAf + 1.0f, fmaf(LA, ed + 1.1920929e-7f, 4.7683716e-7f) + epsA + 1.8e-7f,
                                                    1e-6f);
                            }
                            if (fl & 2u) {
                                epsB = ed + 3.1e-7f;
                                sBfo = pbf * (1.0f / 127.0f);
                                sBexact = false;
                                kB = __frcp_rn(sBfo) / ss.invSbf;
                                qBf = qof;
                                halfB = 0.5f - fmaf(qBf + 1.0f, ed + 4.7683716e-7f + epsB + 1.2e-7f, 1e-6f);
                            }
                        } else {
                            exact();
                            if (fl & 1u) {
                                sA = scale_call(pa, qo);
                                invA = __double2float_rn(recip_call(sA));
                                qAf = qof;
                                const float LA = 0.6931472f * (1.0f + fmaxf(0.0f, -__log2f(__double2float_rn(sA))));
                                halfA = 0.5f - fmaf(qAf + 1.0f, fmaf(LA, ed + 1.1920929e-7f, 4.7683716e-7f), 1e-6f);
                            }
                            if (fl & 2u) {
                                sB = scale_call(pb, qo);
                                kB = __double2float_rn(recip_call(sB)) / ss.invSbf;
                                qBf = qof;
                                halfB = 0.5f - fmaf(qBf + 1.0f, ed + 4.7683716e-7f, 1e-6f);
                            }
                        }
                        clip = !(df * kB * ss.BSmaxf <= qBf + 0.25f && paf * invA * 1.000001f <= qAf + 0.25f);
                    }
                }
            }
            const float dfb = df * kB;
            const float capA = qAf + 0.25f, capB = qBf + 0.25f;
            unsigned ca[16];  // a_bar codes (>= 0) as integers, b_bar codes as exact f32 integers
            float cb[16];
            float raf[16];    // FS: a_bar codes as exact f32 integers
            bool redo = EXACT || sA < 1e-30;  // ex2.approx.ftz flushes below 2^-126
            const float2* BS2 = reinterpret_cast<const float2*>(ss.BSf);
            auto pass1 = [&](auto clamp) {
                constexpr bool CL = decltype(clamp)::value;
                if constexpr (kDefer)
                    if (tt > 0) emit(tt - 1, fl_prev);  // previous step's output
                float mda = 0.0f, mdb = 0.0f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float2 x2 = __fmul2_rn(f2(df), A2f_at(k));
                    float2 qa2 = __fmul2_rn(make_float2(ex2_approx(x2.x), ex2_approx(x2.y)), f2(invA));
                    if constexpr (CL) {
                        qa2.x = fminf(qa2.x, capA);
                        qa2.y = fminf(qa2.y, capA);
                    }
                    const float2 ta = __fadd2_rn(qa2, f2(12582912.0f));
                    const float2 ra = __fadd2_rn(ta, f2(-12582912.0f));
                    const float2 da = __fadd2_rn(qa2, make_float2(-ra.x, -ra.y));
                    if constexpr (FS) {
                        raf[2 * k] = ra.x;
                        raf[2 * k + 1] = ra.y;
                    } else {
                        ca[2 * k] = __float_as_uint(ta.x) - kMagicBits;
                        ca[2 * k + 1] = __float_as_uint(ta.y) - kMagicBits;
                    }
                    float2 qb2 = __fmul2_rn(f2(dfb), BS2[k]);
                    if constexpr (CL) {
                        qb2.x = fminf(fmaxf(qb2.x, -capB), capB);
                        qb2.y = fminf(fmaxf(qb2.y, -capB), capB);
                    }
                    const float2 tb = __fadd2_rn(qb2, f2(12582912.0f));
                    const float2 rb = __fadd2_rn(tb, f2(-12582912.0f));
                    const float2 db = __fadd2_rn(qb2, make_float2(-rb.x, -rb.y));
                    cb[2 * k] = rb.x;
                    cb[2 * k + 1] = rb.y;
                    mda = fmaxf(mda, fmaxf(fabsf(da.x), fabsf(da.y)));
                    mdb = fmaxf(mdb, fmaxf(fabsf(db.x), fabsf(db.y)));
                }
                redo |= (mda > halfA) | (mdb > halfB);
            };
            if (__any_sync(0xffffffffu, clip)) pass1(std::true_type{});
            else pass1(std::false_type{});
            if (redo) {  // exact f64 codes where the f32 quotient is not certified
                exact();
                if constexpr (FS) exact_scales();
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    const float a2 = (m & 1) ? A2f_at(m >> 1).y : A2f_at(m >> 1).x;
                    const float qa_f = fminf(ex2_approx(df * a2) * invA, capA);
                    if (EXACT || sA < 1e-30 || fabsf(qa_f - rintf(qa_f)) > halfA) {
                        const double cq = qdiv_call(exp_call(dmul(delta, arow[m])), sA, static_cast<double>(qAf));
                        ca[m] = static_cast<unsigned>(static_cast<int>(cq));
                        raf[m] = static_cast<float>(cq);
                    }
                    const float qb_f = fminf(fmaxf(dfb * ss.BSf[m], -capB), capB);
                    if (EXACT || fabsf(qb_f - rintf(qb_f)) > halfB)
                        cb[m] = static_cast<float>(qdiv_call(dmul(delta, ss.B[m]), sB, static_cast<double>(qBf)));
                }
            }
            if constexpr (FS) {
                // f32 state update with a rigorous bound (header comment of k3_scan_c1<FS>):
                // P1 = (ra * rh_prev) * f32(S_a S_h'), P2 = rb * f32(S_b u), hf = P1 + P2 stands for
                // h = fl64(fl64(a_q h') + fl64(b_q u)) within D = (max|P1| + max|P2|) 5.2 2^-24
                const float sAf = (fl & 1u) ? sAfo : ss.Saf;
                const float sBf = (fl & 2u) ? sBfo : ss.Sbf;
                const float sAsH = sAf * sHf_prev, sBu = sBf * __double2float_rn(uv);
                float2 hf2[8];
                float phf = 0.0f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float2 p1 = __fmul2_rn(__fmul2_rn(make_float2(raf[2 * k], raf[2 * k + 1]), rhp[k]), f2(sAsH));
                    const float2 p2 = __fmul2_rn(make_float2(cb[2 * k], cb[2 * k + 1]), f2(sBu));
                    const float2 hv = __fadd2_rn(p1, p2);
                    phf = fmaxf(phf, fmaxf(fabsf(hv.x), fabsf(hv.y)));
                    hf2[k] = hv;
                }
                // |P1| <= qA qH' |f32(S_a) f32(S_h')| and |P2| <= qB |f32(S_b) f32(u)| (codes are clipped
                // to their q): D from the step's scalars, with 5.3 u for the rounding of these products
                // (outlier a / b scales: + their relative bound epsA / epsB)
                const float maxD =
                    fmaf(qAf * qHp * sAsH, 5.3f * 5.9604645e-8f + epsA, fmaf(qBf * fabsf(sBu), 5.3f * 5.9604645e-8f + epsB, 1e-37f));
                double sH = ss.Sh, qH = qa;
                float invHf = ss.invShf;
                // exact state path: h-outlier channels (their scale needs the exact peak), peaks
                // not certainly below theta, non-finite values, uncertified codes
                bool hexact = EXACT || !(maxD < 1e30f);
                if (dyn) hexact |= (fl & 4u) || !(fmaf(maxD, 1.0000003f, phf) < thHlo);
                const float capH = qaf + 0.25f;
                const float halfH = 0.5f - fmaf(maxD, invHf * 1.0001f, fmaf(qaf + 1.0f, 1.25e-7f, 1e-6f));
                float chd[16];
                float mdh = 0.0f;
                auto hcodes = [&](auto clamp) {
                    constexpr bool CL = decltype(clamp)::value;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        float2 q = __fmul2_rn(hf2[k], f2(invHf));
                        if constexpr (CL) {
                            q.x = fminf(fmaxf(q.x, -capH), capH);
                            q.y = fminf(fmaxf(q.y, -capH), capH);
                        }
                        const float2 th = __fadd2_rn(q, f2(12582912.0f));
                        const float2 rh = __fadd2_rn(th, f2(-12582912.0f));
                        const float2 dh = __fadd2_rn(q, make_float2(-rh.x, -rh.y));
                        chd[2 * k] = rh.x;
                        chd[2 * k + 1] = rh.y;
                        mdh = fmaxf(mdh, fmaxf(fabsf(dh.x), fabsf(dh.y)));
                    }
                };
                if (__all_sync(0xffffffffu, phf * invHf <= capH)) hcodes(std::false_type{});
                else hcodes(std::true_type{});
                hexact |= !(mdh <= halfH);
                if (hexact) {  // the exact f64 update (ssm.cpp:165-167) and the c1 h logic on it
                    exact_scales();
                    double hn[16];
#pragma unroll
                    for (int m = 0; m < 16; ++m) {
                        const double a_q = dmul(static_cast<double>(raf[m]), sA);
                        const double b_q = dmul(static_cast<double>(cb[m]), sB);
                        const double hp = dmul(static_cast<double>((m & 1) ? rhp[m >> 1].y : rhp[m >> 1].x), sHp);
                        hn[m] = dadd(dmul(a_q, hp), dmul(b_q, uv));
                    }
                    if (dyn) {
                        double ph = 0.0;
#pragma unroll
                        for (int m = 0; m < 16; ++m) ph = fmax(ph, fabs(hn[m]));
                        if (ph > thH) fl |= 4u;
                        if (fl & 4u) {
                            sH = scale_call(ph, qo);
                            invHf = __double2float_rn(recip_call(sH));
                            qH = qo;
                        }
                    }
                    const float qHf = static_cast<float>(qH), capHx = qHf + 0.25f;
                    const float halfHx = 0.5f - fmaf(qHf + 1.0f, 2.3841858e-7f, 1e-6f);
#pragma unroll
                    for (int m = 0; m < 16; ++m) {  // |dq| <= |q| 4 2^-24 from the exact value
                        const float q = fminf(fmaxf(__double2float_rn(hn[m]) * invHf, -capHx), capHx);
                        const float r = rintf(q);
                        chd[m] = (EXACT || !(fabsf(q - r) <= halfHx)) ? static_cast<float>(qdiv_call(hn[m], sH, qH)) : r;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) rhp[k] = make_float2(chd[2 * k], chd[2 * k + 1]);  // carried state
                sHp = sH;
                sHf_prev = (fl & 4u) ? __double2float_rn(sH) : ss.Shf;
                qHp = static_cast<float>(qH);
            } else {
            // pass 2: dequantized values (code * s) and the exact f64 update, ssm.cpp:165-167
                const double nKA = dmul(sA, -4503599627370496.0);
    #pragma unroll
                for (int m = 0; m < 16; ++m) {
                    const double a_q = __fma_rn(__hiloint2double(0x43300000, static_cast<int>(ca[m])), sA, nKA);
                    const double b_q = dmul(static_cast<double>(cb[m]), sB);
                    h[m] = dadd(dmul(a_q, h[m]), dmul(b_q, uv));
                }
                // h detection + codes (see k3_scan_fast): f32 peak = fl32 of the exact peak
                float2 hfv[8];
                float phf = 0.0f;
    #pragma unroll
                for (int k = 0; k < 8; ++k) {
                    hfv[k] = make_float2(__double2float_rn(h[2 * k]), __double2float_rn(h[2 * k + 1]));
                    phf = fmaxf(phf, fmaxf(fabsf(hfv[k].x), fabsf(hfv[k].y)));
                }
                double sH = ss.Sh, qH = qa;
                float invHf = ss.invShf;
                if (dyn && ((fl & 4u) | (phf >= thHf))) {
                    if (!(fl & 4u)) {
                        if (phf > thHf) {
                            fl |= 4u;
                        } else {  // phf == fl32(theta): the exact peak decides
                            double ph = 0.0;
    #pragma unroll
                            for (int m = 0; m < 16; ++m) ph = fmax(ph, fabs(h[m]));
                            if (ph > thH) fl |= 4u;
                        }
                    }
                    if (fl & 4u) {
                        double ph = 0.0;
    #pragma unroll
                        for (int m = 0; m < 16; ++m) ph = fmax(ph, fabs(h[m]));
                        sH = scale_call(ph, qo);
                        invHf = __double2float_rn(recip_call(sH));
                        qH = qo;
                    }
                }
                {  // |dq| <= |q| 4 2^-24 (h and 1/s rounded to f32, one product)
                    const float qHf = static_cast<float>(qH), capH = qHf + 0.25f;
                    const float halfH = 0.5f - fmaf(qHf + 1.0f, 2.3841858e-7f, 1e-6f);
                    float chd[16];
                    bool hredo = EXACT;
                    auto hcodes = [&](auto clamp) {
                        constexpr bool CL = decltype(clamp)::value;
                        float mdh = 0.0f;
    #pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            float2 q = __fmul2_rn(hfv[k], f2(invHf));
                            if constexpr (CL) {
                                q.x = fminf(fmaxf(q.x, -capH), capH);
                                q.y = fminf(fmaxf(q.y, -capH), capH);
                            }
                            const float2 th = __fadd2_rn(q, f2(12582912.0f));
                            const float2 rh = __fadd2_rn(th, f2(-12582912.0f));
                            const float2 dh = __fadd2_rn(q, make_float2(-rh.x, -rh.y));
                            chd[2 * k] = rh.x;
                            chd[2 * k + 1] = rh.y;
                            mdh = fmaxf(mdh, fmaxf(fabsf(dh.x), fabsf(dh.y)));
                        }
                        hredo |= mdh > halfH;
                    };
                    if (__all_sync(0xffffffffu, phf * invHf <= capH)) hcodes(std::false_type{});
                    else hcodes(std::true_type{});
                    if (hredo) {
    #pragma unroll
                        for (int m = 0; m < 16; ++m) {
                            const float hv = (m & 1) ? hfv[m >> 1].y : hfv[m >> 1].x;
                            const float q = fminf(fmaxf(hv * invHf, -capH), capH);
                            if (EXACT || fabsf(q - rintf(q)) > halfH) chd[m] = static_cast<float>(qdiv_call(h[m], sH, qH));
                        }
                    }
    #pragma unroll
    #pragma unroll
                    for (int m = 0; m < 16; ++m) h[m] = dmul(static_cast<double>(chd[m]), sH);  // carried state
                }
            }
            if constexpr (!kDefer) emit(tt, fl);
            fl_prev = fl;
        }
        if constexpr (kDefer) emit(nt - 1, fl_prev);
    }
    if constexpr (MT) {
        // the last of the directions to finish this (sample, group) quantizes its merged output
        const size_t ci = static_cast<size_t>(s) * (gridDim.x / P.n) + grp;
        __threadfence();  // this warp's o stores are visible before its arrival
        int prev = 0;
        if (lane == 0) prev = atomicAdd(P.merge_cnt + ci, 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev != P.n - 1) return;
        if (lane == 0) P.merge_cnt[ci] = 0;  // ready for the next launch
        __threadfence();
        merge_tail(P.merge, s, grp, lane);
    }
}

// Shapes measured at Vim-B batch 256 (ms per launch, both directions): one warp
// per CTA, 4-step chunks, 12 CTAs per SM (<= 168 registers) 2.225; two or four
// warps per CTA 2.306 / 2.375; 8-step chunks 2.376; 128 registers (16 warps per SM)
// spills and runs 3.01; per-lane cp.async staging instead of bulk rows 2.306.
constexpr int kC1Chunk = 4, kC1MinBlocks = 12;

template <bool EXACT, int ABITS, bool TRACE, bool FS, int MB = kC1MinBlocks, bool SMA2 = false, bool MT = false>
static cudaError_t launch_c1(const ScanDirs& P, int ndirs, const StepShared* steps, cudaStream_t st) {
    constexpr auto kern = k3_scan_c1<EXACT, ABITS, TRACE, kC1Chunk, MB, FS, SMA2, MT>;
    const int smem = static_cast<int>(sizeof(C1Smem<kC1Chunk>));
    cudaError_t e = ensure_smem_attr<kern>(smem);
    if (e != cudaSuccess) return e;
    dim3 grid(((P.d[0].E + 31) / 32) * ndirs, P.d[0].S, 1);
    kern<<<grid, 32, smem, st>>>(P, steps);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

template <bool EXACT, int ABITS, bool TRACE, bool FS = false>
static cudaError_t launch_fast(const ScanDirs& P, int ndirs, const StepShared* steps, cudaStream_t st) {
    const int smem = static_cast<int>(sizeof(WarpSmem)) * (kThr / 32);
    cudaError_t e = ensure_smem_attr<k3_scan_fast<EXACT, ABITS, TRACE, FS>>(smem);
    if (e != cudaSuccess) return e;
    dim3 grid((P.d[0].E + kCh - 1) / kCh, P.d[0].S, ndirs);
    k3_scan_fast<EXACT, ABITS, TRACE, FS><<<grid, kThr, smem, st>>>(P, steps);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

// kernel: 0 the one-thread-per-channel kernel (needs an even E: 16-byte rows), 1 the
// two-threads-per-channel kernel, 2 the one-thread-per-channel kernel with the f32 state update
template <int ABITS, bool FS>
static cudaError_t launch_c1_any(const ScanDirs& P, int ndirs, const StepShared* steps, cudaStream_t st, bool exact,
                                 bool trace, bool force_big = false) {
    if (exact) return trace ? launch_c1<true, ABITS, true, FS>(P, ndirs, steps, st) : launch_c1<true, ABITS, false, FS>(P, ndirs, steps, st);
    if (trace) return launch_c1<false, ABITS, true, FS>(P, ndirs, steps, st);
    // FS on large grids (>= 2 waves of 16 CTAs per SM): A stays in shared memory and the
    // kernel fits 128 registers, 16 warps per SM (Vim-B batch 256: 1.705 vs 1.741 ms); small
    // grids keep 168 registers (Vim-S batch 64: 0.286 vs 0.296)
    const long ctas = static_cast<long>((P.d[0].E + 31) / 32) * P.d[0].S * ndirs;
    const bool big = force_big || ctas >= 2L * 148 * 16;
    if (FS && P.merge_cnt) {
        if (big) return launch_c1<false, ABITS, false, FS, 13, true, true>(P, ndirs, steps, st);
        return launch_c1<false, ABITS, false, FS, kC1MinBlocks, false, true>(P, ndirs, steps, st);
    }
    if (FS && big) return launch_c1<false, ABITS, false, FS, 13, true>(P, ndirs, steps, st);
    return launch_c1<false, ABITS, false, FS>(P, ndirs, steps, st);
}

template <int ABITS>
static cudaError_t launch_kernel(const ScanDirs& P, int ndirs, const StepShared* steps, cudaStream_t st,
                                 int kernel, bool exact, bool trace, bool force_big = false) {
    if (kernel == 0) return launch_c1_any<ABITS, false>(P, ndirs, steps, st, exact, trace);
    if (kernel == 2) return launch_c1_any<ABITS, true>(P, ndirs, steps, st, exact, trace, force_big);
    if (kernel == 3) {  // two threads per channel, f32 state update
        if (exact) return trace ? launch_fast<true, ABITS, true, true>(P, ndirs, steps, st) : launch_fast<true, ABITS, false, true>(P, ndirs, steps, st);
        return trace ? launch_fast<false, ABITS, true, true>(P, ndirs, steps, st) : launch_fast<false, ABITS, false, true>(P, ndirs, steps, st);
    }
    if (exact) return trace ? launch_fast<true, ABITS, true>(P, ndirs, steps, st) : launch_fast<true, ABITS, false>(P, ndirs, steps, st);
    return trace ? launch_fast<false, ABITS, true>(P, ndirs, steps, st) : launch_fast<false, ABITS, false>(P, ndirs, steps, st);
}

// ---- small batches: the scan split into three phases -----------------------------
// At batch 1 (BASELINE C1) a launch has a few warps on the whole GPU, so each step
// costs its full instruction latency. Only the h update is sequential in t; the
// a_bar / b_bar codes (their detector state runs per refresh window) and the output
// sum are not. So: (A) codes for every (step, channel) — detection per (step,
// channel), the sticky state per channel, codes on sixteen lanes per channel
// (k3s_codes16); (B) the f32 state update (k3_scan_c1<FS>) walking the steps on
// sixteen lanes per channel, one state each (k3s_state16); (C) the outputs of every
// (step, channel) in parallel (k3s_out). Same arithmetic as k3_scan_c1<FS>; the
// intermediates (88 B per direction, sample, step and channel) stay in L2 at these
// sizes.
// phase A's record per (direction, sample, step, channel): a_bar codes (0..q) | b_bar codes |
// the exact scales of the step (outlier channels: their own) | outlier flags after detection
// plus the f32 scalars phase B's common path needs: f32 of the a scale, f32(S_b) f32(u)
// and q_b |that| (k3_scan_c1<FS>'s sAf, sBu and the b term of its bound D)
struct __align__(16) SmallRec {
    uint4 ca, cb;
    double sA, sB;
    unsigned fab;
    float sAf, sBu, qBsBu;
};
static_assert(sizeof(SmallRec) == 64, "four 16-byte copies per record");
struct SmallWork {
    SmallRec* rec;  // [dir][s][t][E]
    int8_t* rh;     // [dir][s][t][E][16] h codes
    double* sh;     // [dir][s][t][E] h scale
};
constexpr size_t kSmallPerElem = sizeof(SmallRec) + 16 + 8;
constexpr long kSmallMaxChannels = 148L * 32;  // below one warp per SM: the split path

static bool small_path(int S, int E, int ndirs) {
    return static_cast<long>(S) * E * ndirs <= kSmallMaxChannels && (E % 32) == 0;
}

static SmallWork small_work(void* base, int S, int T, int E, int ndirs) {
    const size_t n = static_cast<size_t>(ndirs) * S * T * E;
    uint8_t* q = static_cast<uint8_t*>(base);
    SmallWork w;
    w.rec = reinterpret_cast<SmallRec*>(q);
    q += n * sizeof(SmallRec);
    w.rh = reinterpret_cast<int8_t*>(q);
    q += n * 16;
    w.sh = reinterpret_cast<double*>(q);
    return w;
}

constexpr int kSA = 16;  // steps staged per pass of phase A
// (A') one CTA per (8 channels, refresh window). The channel's detector is split into
// its independent parts: per (step, channel) the certified delta / peaks and the
// detection of that step (exact where the f32 peak is within its bound of theta); the
// sticky O state is a prefix OR along the window (maybe_refresh clears it), one thread
// per channel; then per (step, channel) the step's scales and margins (outlier
// channels' exact scales); then sixteen lanes per channel, lane m computing state m's
// a_bar / b_bar codes from those. Same values as k3_scan_c1's per-step detector (the
// OR of the per-step detections equals its sticky update, which skips the test once a
// bit is set). The window's step records and inputs are staged per pass of kSA steps.
struct SmallStepScal {  // per (step, channel)
    float df, invA, dfb, halfA, halfB;
    unsigned fl;
    double sA, sB;
};
constexpr int kCh16 = 8;  // channels per CTA of the sixteen-lane phases (128 threads)
struct SmallA16Smem {
    StepShared st[kSA];
    double dp[kSA][kCh16];
    double u[kSA][kCh16];
    SmallStepScal sc[kSA][kCh16];
    unsigned char det[kSA][kCh16];
    double amax[kCh16], bd[kCh16];
};

template <int ABITS>
__global__ void __launch_bounds__(128) k3s_codes16(const ScanDirs P, const StepShared* __restrict__ steps, SmallWork w,
                                                   int win) {
    extern __shared__ __align__(16) uint8_t sa16_smem_raw[];
    SmallA16Smem& sm = *reinterpret_cast<SmallA16Smem*>(sa16_smem_raw);
    const int ndirs = P.n;
    const int nwin = (P.d[0].T + win - 1) / win;
    const int dir = static_cast<int>(blockIdx.y) % ndirs, sw = static_cast<int>(blockIdx.y) / ndirs;
    const ScanParams& p = P.d[dir];
    const int tid = threadIdx.x, cl = tid >> 4, m = tid & 15;
    const int E = p.E, T = p.T, P2 = E + 32, ch0 = static_cast<int>(blockIdx.x) * kCh16, i = ch0 + cl;
    const int s = sw / nwin;
    const int t0 = (sw % nwin) * win, t1 = min(T, t0 + win);
    const bool dyn = p.mode == MODE_DYNAMIC;
    constexpr double qa = static_cast<double>((1 << (ABITS - 1)) - 1), qo = 127.0;
    constexpr float qaf = static_cast<float>(qa), qof = 127.0f;
    const double am = p.a[static_cast<size_t>(i) * 16 + m];
    const float A2m = __double2float_rn(am * 1.4426950408889634);
    if (tid < kCh16) {
        const double* arow = p.a + static_cast<size_t>(ch0 + tid) * 16;
        double Amax = -1e300;
#pragma unroll
        for (int k = 0; k < 16; ++k) Amax = fmax(Amax, arow[k]);
        sm.amax[tid] = Amax;
        sm.bd[tid] = p.b_delta[ch0 + tid];
    }
    const double thA = p.cal[0].theta, thB = p.cal[1].theta;
    const float thAf = __double2float_rn(thA), thBf = __double2float_rn(thB);
    const size_t rowbase = static_cast<size_t>(dir) * p.S * T + static_cast<size_t>(s) * T;
    constexpr int kStPieces = static_cast<int>(sizeof(StepShared) / 16);
    unsigned flc = 0;  // threads < kCh16: channel tid's O state along the window
    for (int tb = t0; tb < t1; tb += kSA) {
        const int nt = min(kSA, t1 - tb);
        __syncthreads();  // the previous pass is consumed
        for (int q = tid; q < nt * kStPieces; q += 128) {
            const int tt = q / kStPieces, k = q % kStPieces;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(
                             reinterpret_cast<uint4*>(&sm.st[tt]) + k)),
                         "l"(reinterpret_cast<const uint4*>(steps + rowbase + tb + tt) + k) : "memory");
        }
        for (int q = tid; q < nt * kCh16; q += 128) {
            const int tt = q / kCh16, c = q % kCh16;
            cp_async8(&sm.dp[tt][c], p.proj + (static_cast<size_t>(s) * T + tb + tt) * P2 + ch0 + c, true);
            cp_async8(&sm.u[tt][c], p.u + (static_cast<size_t>(s) * T + row_at(p.order, tb + tt, T, p.grid)) * E + ch0 + c,
                      true);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        // (1) per (step, channel): this step's detection (detect_outliers, channel-local form)
        if (dyn) {
            for (int q = tid; q < nt * kCh16; q += 128) {
                const int tt = q / kCh16, c = q % kCh16;
                const StepShared& ss = sm.st[tt];
                const double x = dadd(sm.dp[tt][c], sm.bd[c]);  // ssm.cpp:150-151
                float ed;
                const float df = softplus_f32(__double2float_rn(x), ed);
                const float x2m = df * __double2float_rn(sm.amax[c] * 1.4426950408889634);
                const float paf = ex2_approx(x2m);
                const float ea = 2.0f * fmaf(0.6931472f * fabsf(x2m), ed + 1.1920929e-7f, 4.7683716e-7f) + 1e-6f;
                const float pbf = df * ss.Bmaxf;
                const float eb = 2.0f * (ed + 2.3841858e-7f) + 1e-6f;
                unsigned d = 0;
                bool have = false;
                double pa = 0.0, pb = 0.0;
                auto exact = [&]() {
                    if (!have) {
                        const double delta = softplus_call(x);
                        pa = exp_call(dmul(delta, sm.amax[c]));
                        pb = dmul(delta, ss.Bmax);
                        have = true;
                    }
                };
                if (paf > thAf * (1.0f + ea)) {
                    d |= 1u;
                } else if (paf >= thAf * (1.0f - ea)) {
                    exact();
                    if (pa > thA) d |= 1u;
                }
                if (pbf > thBf * (1.0f + eb)) {
                    d |= 2u;
                } else if (pbf >= thBf * (1.0f - eb)) {
                    exact();
                    if (pb > thB) d |= 2u;
                }
                sm.det[tt][c] = static_cast<unsigned char>(d);
            }
            __syncthreads();
            // (2) the sticky O state: maybe_refresh, then the step's detection
            if (tid < kCh16) {
                for (int tt = 0; tt < nt; ++tt) {
                    flc = (flc & static_cast<unsigned>(sm.st[tt].keep)) | sm.det[tt][tid];
                    sm.sc[tt][tid].fl = flc;
                }
            }
        } else {
            for (int q = tid; q < nt * kCh16; q += 128) sm.sc[q / kCh16][q % kCh16].fl = 0u;
        }
        __syncthreads();
        // (3) per (step, channel): scales and margins of the step (outlier channels: their
        // exact scales), and the record's scalars
        for (int q = tid; q < nt * kCh16; q += 128) {
            const int tt = q / kCh16, c = q % kCh16;
            const StepShared& ss = sm.st[tt];
            SmallStepScal& sc = sm.sc[tt][c];
            const unsigned fl = sc.fl;
            const double x = dadd(sm.dp[tt][c], sm.bd[c]);
            float ed;
            const float df = softplus_f32(__double2float_rn(x), ed);
            double sA = ss.Sa, sB = ss.Sb;
            float invA = ss.invSaf, kB = 1.0f;
            float halfA = fmaf(-ss.hA1, ed, ss.hA0);
            float halfB = fmaf(-(qaf + 1.0f), ed, 0.5f - fmaf(qaf + 1.0f, 4.7683716e-7f, 1e-6f));
            if (fl & 3u) {
                const double delta = softplus_call(x);
                if (fl & 1u) {
                    sA = scale_call(exp_call(dmul(delta, sm.amax[c])), qo);
                    invA = __double2float_rn(recip_call(sA));
                    const float LA = 0.6931472f * (1.0f + fmaxf(0.0f, -__log2f(__double2float_rn(sA))));
                    halfA = 0.5f - fmaf(qof + 1.0f, fmaf(LA, ed + 1.1920929e-7f, 4.7683716e-7f), 1e-6f);
                }
                if (fl & 2u) {
                    sB = scale_call(dmul(delta, ss.Bmax), qo);
                    kB = __double2float_rn(recip_call(sB)) / ss.invSbf;
                    halfB = 0.5f - fmaf(qof + 1.0f, ed + 4.7683716e-7f, 1e-6f);
                }
            }
            sc.df = df;
            sc.invA = invA;
            sc.dfb = df * kB;
            sc.halfA = halfA;
            sc.halfB = halfB;
            sc.sA = sA;
            sc.sB = sB;
            SmallRec& rec = w.rec[(rowbase + tb + tt) * E + ch0 + c];
            rec.sA = sA;
            rec.sB = sB;
            rec.fab = fl;
            const float sBu = ((fl & 2u) ? __double2float_rn(sB) : ss.Sbf) * __double2float_rn(sm.u[tt][c]);
            rec.sAf = (fl & 1u) ? __double2float_rn(sA) : ss.Saf;
            rec.sBu = sBu;
            rec.qBsBu = ((fl & 2u) ? qof : qaf) * fabsf(sBu);
        }
        __syncthreads();
        // (4) sixteen lanes per channel: state m's clamped quotients (k3_scan_c1's clamp
        // form), exact where uncertified
        for (int tt = 0; tt < nt; ++tt) {
            const StepShared& ss = sm.st[tt];
            const SmallStepScal& sc = sm.sc[tt][cl];
            const unsigned fl = sc.fl;
            const float qAf = (fl & 1u) ? qof : qaf, qBf = (fl & 2u) ? qof : qaf;
            const float capA = qAf + 0.25f, capB = qBf + 0.25f;
            int ca, cb;
            const float qaq = fminf(ex2_approx(sc.df * A2m) * sc.invA, capA);
            const float ra = rintf(qaq);
            if (sc.sA < 1e-30 || !(fabsf(qaq - ra) <= sc.halfA)) {  // ex2.approx.ftz flushes below 2^-126
                const double delta = softplus_call(dadd(sm.dp[tt][cl], sm.bd[cl]));
                ca = static_cast<int>(qdiv_call(exp_call(dmul(delta, am)), sc.sA, static_cast<double>(qAf)));
            } else {
                ca = static_cast<int>(ra);
            }
            const float qbq = fminf(fmaxf(sc.dfb * ss.BSf[m], -capB), capB);
            const float rb = rintf(qbq);
            if (!(fabsf(qbq - rb) <= sc.halfB)) {
                const double delta = softplus_call(dadd(sm.dp[tt][cl], sm.bd[cl]));
                cb = static_cast<int>(qdiv_call(dmul(delta, ss.B[m]), sc.sB, static_cast<double>(qBf)));
            } else {
                cb = static_cast<int>(rb);
            }
            SmallRec& rec = w.rec[(rowbase + tb + tt) * E + i];
            reinterpret_cast<int8_t*>(&rec.ca)[m] = static_cast<int8_t>(ca);
            reinterpret_cast<int8_t*>(&rec.cb)[m] = static_cast<int8_t>(cb);
        }
    }
}

__device__ __forceinline__ void unpack_codes16(uint4 v, float (&c)[16]) {
    const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int m = 0; m < 16; ++m) c[m] = static_cast<float>(static_cast<int8_t>(wd[m >> 2] >> (8 * (m & 3))));
}

// (B') sixteen lanes per channel, lane m owning state m: the same update with the
// per-channel decisions as group votes. phf <= theta' and max|d| <= half hold iff they
// hold on every lane (fl32(x + a) is monotone in x; fmaxf(0, .) keeps the NaN rule of
// the max chain), so the group's ballot decides the exact path exactly as (B) does; the
// exact path's peak is a 16-lane max (shuffles within the group). A step's critical path
// is then a handful of dependent f32 ops and one vote instead of 16 states in series.
constexpr int kSB16 = 8;   // steps per staged chunk
struct SmallB16Smem {
    SmallRec rec[2][kSB16][kCh16];
    double u[2][kSB16][kCh16];
    StepShared st[2][kSB16];
};

template <int ABITS>
__global__ void __launch_bounds__(128) k3s_state16(const ScanDirs P, const StepShared* __restrict__ steps,
                                                   SmallWork w) {
    extern __shared__ __align__(16) uint8_t sb16_smem_raw[];
    SmallB16Smem& sh = *reinterpret_cast<SmallB16Smem*>(sb16_smem_raw);
    const int ndirs = P.n;
    const int dir = static_cast<int>(blockIdx.y) % ndirs, s = static_cast<int>(blockIdx.y) / ndirs;
    const ScanParams& p = P.d[dir];
    const int tid = threadIdx.x, lane = tid & 31, cl = tid >> 4, m = tid & 15;
    const int E = p.E, T = p.T, ch0 = static_cast<int>(blockIdx.x) * kCh16, i = ch0 + cl;
    const unsigned gmask = 0xFFFFu << (lane & 16);
    const bool dyn = p.mode == MODE_DYNAMIC;
    constexpr double qa = static_cast<double>((1 << (ABITS - 1)) - 1), qo = 127.0;
    constexpr float qaf = static_cast<float>(qa);
    const double thH = p.cal[2].theta;
    const float thHlo = __double2float_rn(thH) * (1.0f - 4.0f * 5.9604645e-8f);
    const size_t rowbase = static_cast<size_t>(dir) * p.S * T + static_cast<size_t>(s) * T;
    constexpr int kStPieces = static_cast<int>(sizeof(StepShared) / 16);
    auto issue = [&](int t0, int buf) {  // records, scan inputs and step records of chunk t0 (16-byte copies)
        for (int q = tid; q < kSB16 * kCh16 * 4; q += 128) {
            const int tt = q / (kCh16 * 4), c = (q / 4) % kCh16, k = q % 4;
            const int t = min(t0 + tt, T - 1);
            const uint4* src = reinterpret_cast<const uint4*>(w.rec + (rowbase + t) * E + ch0 + c) + k;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(
                             reinterpret_cast<uint4*>(&sh.rec[buf][tt][c]) + k)), "l"(src) : "memory");
        }
        for (int q = tid; q < kSB16 * kCh16; q += 128) {
            const int tt = q / kCh16, c = q % kCh16;
            const int t = min(t0 + tt, T - 1);
            cp_async8(&sh.u[buf][tt][c], p.u + (static_cast<size_t>(s) * T + row_at(p.order, t, T, p.grid)) * E + ch0 + c,
                      true);
        }
        for (int q = tid; q < kSB16 * kStPieces; q += 128) {
            const int tt = q / kStPieces, k = q % kStPieces;
            const int t = min(t0 + tt, T - 1);
            const uint4* src = reinterpret_cast<const uint4*>(steps + rowbase + t) + k;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(
                             reinterpret_cast<uint4*>(&sh.st[buf][tt]) + k)), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float rhp = 0.0f;  // this state's previous code (exact f32 integer)
    double sHp = 0.0;
    float sHf_prev = 0.0f, qHp = 0.0f;
    unsigned flh = 0;
    issue(0, 0);
    for (int t0 = 0, ci = 0; t0 < T; t0 += kSB16, ++ci) {
        const int nt = min(kSB16, T - t0), cur = ci & 1;
        if (t0 + kSB16 < T) {
            issue(t0 + kSB16, cur ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        // the step's inputs that do not depend on the carried state, loaded (and the next
        // step's prefetched) ahead of the carried chain so the in-order issue overlaps them
        struct In {
            float raf, cbf, sAf, sBu, qBsBu, qAf, invHf, Shf;
            double Sh;
            unsigned keep;
        };
        auto load = [&](int tt) {
            In v;
            const StepShared& ss = sh.st[cur][tt];
            const SmallRec& r = sh.rec[cur][tt][cl];
            v.raf = static_cast<float>(reinterpret_cast<const int8_t*>(&r.ca)[m]);
            v.cbf = static_cast<float>(reinterpret_cast<const int8_t*>(&r.cb)[m]);
            const float4 f = *reinterpret_cast<const float4*>(&r.fab);  // fab | sAf | sBu | qBsBu
            v.qAf = (__float_as_uint(f.x) & 1u) ? 127.0f : qaf;
            v.sAf = f.y;
            v.sBu = f.z;
            v.qBsBu = f.w;
            v.keep = static_cast<unsigned>(ss.keep);
            v.Sh = ss.Sh;
            v.invHf = ss.invShf;
            v.Shf = ss.Shf;
            return v;
        };
        int8_t* rh_out = w.rh + ((rowbase + t0) * E + i) * 16 + m;
        double* sh_out = w.sh + (rowbase + t0) * E + i;
        In cu = load(0);
#pragma unroll 1
        for (int tt = 0; tt < nt; ++tt, rh_out += static_cast<size_t>(E) * 16, sh_out += E) {
            if (dyn) flh &= cu.keep & 4u;
            const float sAsH = cu.sAf * sHf_prev;
            const float hv = __fadd_rn(__fmul_rn(__fmul_rn(cu.raf, rhp), sAsH), __fmul_rn(cu.cbf, cu.sBu));
            const float maxD = fmaf(fmaf(cu.qAf * qHp, sAsH, cu.qBsBu), 5.3f * 5.9604645e-8f, 1e-37f);
            double sH = cu.Sh, qH = qa;
            float invHf = cu.invHf;
            const float capH = qaf + 0.25f;
            const float halfH = 0.5f - fmaf(maxD, invHf * 1.0001f, fmaf(qaf + 1.0f, 1.25e-7f, 1e-6f));
            const float q = fminf(fmaxf(__fmul_rn(hv, invHf), -capH), capH);
            float chd = rintf(q);
            bool bad = !(fabsf(q - chd) <= halfH) || !(maxD < 1e30f);
            if (dyn) bad |= (flh & 4u) || !(fmaf(maxD, 1.0000003f, fmaxf(0.0f, fabsf(hv))) < thHlo);
            const In nx = load(tt + 1 < nt ? tt + 1 : tt);
            if (__ballot_sync(0xffffffffu, bad) & gmask) {  // the channel's exact f64 update
                const SmallRec& r = sh.rec[cur][tt][cl];
                const double a_q = dmul(static_cast<double>(cu.raf), r.sA);
                const double b_q = dmul(static_cast<double>(cu.cbf), r.sB);
                const double hn = dadd(dmul(a_q, dmul(static_cast<double>(rhp), sHp)), dmul(b_q, sh.u[cur][tt][cl]));
                if (dyn) {
                    double ph = fabs(hn);
#pragma unroll
                    for (int o = 8; o >= 1; o >>= 1) ph = fmax(ph, __shfl_xor_sync(gmask, ph, o));
                    if (ph > thH) flh |= 4u;
                    if (flh & 4u) {
                        sH = scale_call(ph, qo);
                        invHf = __double2float_rn(recip_call(sH));
                        qH = qo;
                    }
                }
                const float qHf = static_cast<float>(qH), capHx = qHf + 0.25f;
                const float halfHx = 0.5f - fmaf(qHf + 1.0f, 2.3841858e-7f, 1e-6f);
                const float qx = fminf(fmaxf(__double2float_rn(hn) * invHf, -capHx), capHx);
                const float rr = rintf(qx);
                chd = !(fabsf(qx - rr) <= halfHx) ? static_cast<float>(qdiv_call(hn, sH, qH)) : rr;
            }
            *rh_out = static_cast<int8_t>(static_cast<int>(chd));
            if (m == 0) *sh_out = sH;
            rhp = chd;
            sHp = sH;
            sHf_prev = (flh & 4u) ? __double2float_rn(sH) : cu.Shf;
            qHp = static_cast<float>(qH);
            cu = nx;
        }
        __syncthreads();  // chunk consumed before its buffer is refilled
    }
}

// (C) one thread per (direction, sample, step, channel): o = 0 + C_0 h_0 + ... + C_15 h_15
// with h = code * scale (ssm.cpp:170-174), stored at the canonical row
__global__ void __launch_bounds__(256) k3s_out(const ScanDirs P, const StepShared* __restrict__ steps, SmallWork w) {
    const ScanParams& p0 = P.d[0];
    const int E = p0.E, T = p0.T, S = p0.S;
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t n = static_cast<size_t>(P.n) * S * T * E;
    if (idx >= n) return;
    const int i = static_cast<int>(idx % E);
    const size_t row = idx / E;  // (dir * S + s) * T + t
    const int dir = static_cast<int>(row / (static_cast<size_t>(S) * T));
    const int s = static_cast<int>((row / T) % S);
    const StepShared& ss = steps[row];
    float rc[16];
    unpack_codes16(reinterpret_cast<const uint4*>(w.rh)[idx], rc);
    const double sH = w.sh[idx];
    double o = 0.0;
#pragma unroll
    for (int m = 0; m < 16; ++m) o = dadd(o, dmul(ss.C[m], dmul(static_cast<double>(rc[m]), sH)));
    P.d[dir].o[static_cast<size_t>(s) * T * E + ss.ocol + i] = o;
}

template <int ABITS>
static cudaError_t launch_small(const ScanDirs& P, int ndirs, const StepShared* steps, void* small_base,
                                cudaStream_t st) {
    const ScanParams& p = P.d[0];
    const SmallWork w = small_work(small_base, p.S, p.T, p.E, ndirs);
    const bool dyn = p.mode == MODE_DYNAMIC;
    // refresh windows carry the a_bar / b_bar detector state; without refreshes it runs
    // through the whole sequence (static mode has none: any window)
    const int win = dyn ? (p.n_refresh > 0 ? p.n_refresh : p.T) : 8;
    const int nwin = (p.T + win - 1) / win;
    cudaError_t ea = ensure_smem_attr<k3s_codes16<ABITS>>(static_cast<int>(sizeof(SmallA16Smem)));
    if (ea != cudaSuccess) return ea;
    k3s_codes16<ABITS><<<dim3(p.E / kCh16, p.S * nwin * ndirs), 128, sizeof(SmallA16Smem), st>>>(P, steps, w, win);
    ++kernel_launch_counter();
    cudaError_t e = ensure_smem_attr<k3s_state16<ABITS>>(static_cast<int>(sizeof(SmallB16Smem)));
    if (e != cudaSuccess) return e;
    k3s_state16<ABITS><<<dim3(p.E / kCh16, p.S * ndirs), 128, sizeof(SmallB16Smem), st>>>(P, steps, w);
    ++kernel_launch_counter();
    const size_t n = static_cast<size_t>(ndirs) * p.S * p.T * p.E;
    k3s_out<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(P, steps, w);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

size_t scan_fast_workspace_bytes(int S, int T, int ndirs, int E) {
    const size_t steps = static_cast<size_t>(ndirs) * S * T * sizeof(StepShared);
    return steps + ((E > 0 && small_path(S, E, ndirs)) ? static_cast<size_t>(ndirs) * S * T * E * kSmallPerElem : 0);
}

cudaError_t launch_scan_fast(const ScanParams* dirs, int ndirs, void* work, size_t work_bytes, cudaStream_t st,
                             int variant, const K1Params* merge, int* merge_cnt, bool* merged) {
    if (merged) *merged = false;
    if (ndirs < 1 || ndirs > 2) return cudaErrorInvalidValue;
    ScanDirs P;
    P.n = ndirs;
    for (int k = 0; k < ndirs; ++k) {
        P.d[k] = dirs[k];
        if (dirs[k].N != 16 || dirs[k].E != dirs[0].E || dirs[k].S != dirs[0].S || dirs[k].T != dirs[0].T)
            return cudaErrorInvalidValue;
        if (dirs[k].mode != MODE_DYNAMIC && dirs[k].mode != MODE_STATIC) return cudaErrorInvalidValue;
    }
    if (dirs[0].obits != 8) return cudaErrorNotSupported;  // fast path is built for 8-bit outliers
    if (dirs[0].abits != 4 && dirs[0].abits != 8) return cudaErrorNotSupported;
    const int S = dirs[0].S, T = dirs[0].T;
    if (!work || work_bytes < scan_fast_workspace_bytes(S, T, ndirs, 0) || (reinterpret_cast<uintptr_t>(work) & 15))
        return cudaErrorInvalidValue;
    StepShared* steps = static_cast<StepShared*>(work);
    const int warps = ndirs * T * ((S + kTabSamples - 1) / kTabSamples);
    k3_step_tables<<<(warps + 7) / 8, 256, 0, st>>>(P, ndirs, steps);
    ++kernel_launch_counter();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const bool trace = dirs[0].masks != nullptr;
    const bool even = (dirs[0].E & 1) == 0;
    // auto: one thread per channel with the f32 state update for A4 (ms per Vim-B launch at
    // batch 256: 1.70, vs 2.23 with the f64 state update and 2.43 with two threads per
    // channel; Vim-S batch 64: 0.286 / 0.360 / 0.415), two threads per channel with the f32
    // state update for A8 (Vim-T batch 256: 1.100 vs 1.154 with the f64 state, 1.41 / 1.63
    // one thread per channel; batch 1: 7.22 vs 7.38 ms per forward's 24 scans)
    int kernel = (dirs[0].abits == 4 && even) ? 2 : 3;
    if (variant == 2) kernel = 1;
    if (variant == 3 || variant == 4) {
        if (!even) return cudaErrorNotSupported;
        kernel = variant == 3 ? 0 : 2;
    }
    if (variant == 5) kernel = 1;
    if (variant == 6) {  // the large-grid shape of the f32-state kernel (A in shared memory) at any size
        if (!even) return cudaErrorNotSupported;
        kernel = 2;
    }
    const bool exact = variant == 1;
    // the out_proj input K1 rides on the f32-state kernel's tail (plain, non-trace launches;
    // the caller zeroes ocnt and keeps merge_cnt zero between launches)
    if (merge && merge_cnt && kernel == 2 && !exact && !trace && merge->mode != MODE_FP && merge->src == K1_SRC_MERGE &&
        !merge->force_literal && !merge->scanned && merge->E == dirs[0].E && merge->T == T && merge->S == S &&
        (merge->E % 32) == 0 && (!merge->codes4 || merge->abits == 4)) {
        P.merge = *merge;
        P.merge_cnt = merge_cnt;
        if (merged) *merged = true;
    }
    // small batches (< one warp per SM): the split-phase scan (auto only; it needs the
    // workspace's second part)
    const int E = dirs[0].E;
    if (variant == 0 && !trace && !P.merge_cnt && small_path(S, E, ndirs) &&
        work_bytes >= scan_fast_workspace_bytes(S, T, ndirs, E)) {
        void* small_base = static_cast<uint8_t*>(work) + scan_fast_workspace_bytes(S, T, ndirs, 0);
        return dirs[0].abits == 4 ? launch_small<4>(P, ndirs, steps, small_base, st)
                                  : launch_small<8>(P, ndirs, steps, small_base, st);
    }
    switch (dirs[0].abits) {
        case 4: return launch_kernel<4>(P, ndirs, steps, st, kernel, exact, trace, variant == 6);
        default: return launch_kernel<8>(P, ndirs, steps, st, kernel, exact, trace, variant == 6);
    }
}

}  // namespace ob
