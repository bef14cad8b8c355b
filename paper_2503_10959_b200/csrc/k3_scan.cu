// K3 — quantized S6 selective scan (one direction), fused delta-softplus and
// discretization, in-loop dynamic quantization of a_bar, b_bar and h.
//
// Restates, per scan step t (s6_scan, ssm.cpp:147-175, with the QuantHook
// policy of quant.cpp:467-501):
//   delta_i = softplus(dpre_i + b_delta_i)                    ssm.cpp:150-151
//   a_bar[i,m] = exp(delta_i * A[i,m]); b_bar[i,m] = delta_i * B_m   :154-159
//   QuantHook(a_bar), QuantHook(b_bar)                        :163, quant.cpp:493-497
//   h = a_bar .* h + b_bar .* u_i                             :165-167
//   QuantHook(h)   (the quantized h is the carried state)     :168
//   o_i = sum_m C_m * h[i,m]  (m ascending from 0.0)          :170-174
// dpre/B/C come from the x_proj quant-linear (D2) or the f64 projection.
//
// The recurrence is strictly sequential in t (h is quantized and fed back),
// so parallelism is batch x channel: one thread owns one channel's N=16
// states in registers for the whole scan. The detector is channel-local:
// where C(t) = fl(nextafter(theta,+inf)/q_a) > S^I(t) holds (checked on the
// host per (tensor, t)), detect_outliers' list update equals
// O(t) = (refresh ? {} : O(t-1)) U {ch : peak_ch > theta} exactly
// (DESIGN.md §3.3), so threads never synchronize. Steps where C(t) fails run
// the LITERAL variant: one CTA holds every channel of a (sample, direction)
// and takes the cross-channel max of the reference with a block reduction.
#include "common.cuh"
#include "kernels.h"

namespace ob {

__device__ __forceinline__ double block_max(double v, double* red) {
    v = warp_max(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double m = 0.0;
    for (int k = 0; k < nw; ++k) m = fmax(m, red[k]);
    return m;
}

template <bool LITERAL, int N>
__device__ __forceinline__ void quant_row(double (&x)[N], bool& in, int kind, int t, const ScanParams& p, int i,
                                          bool active, bool lit_step, double qa, double qo, double* red, int s) {
    const ScanKindCal& kc = p.cal[kind];
    double peak = 0.0;
#pragma unroll
    for (int m = 0; m < N; ++m) peak = fmax(peak, fabs(x[m]));
    if (p.mode == MODE_FP) {
        if (kc.peaks && active)
            atomicMax(kc.peaks + static_cast<size_t>(t) * p.E + i,
                      static_cast<unsigned long long>(__double_as_longlong(peak)));
        return;
    }
    if (p.mode == MODE_STATIC) {
        const double S = kc.s_full[t], inv = __ddiv_rn(1.0, S);
#pragma unroll
        for (int m = 0; m < N; ++m) x[m] = dmul(quant_code_inv(x[m], S, inv, qa), S);
        return;
    }
    if (refresh_at(t, p.n_refresh)) in = false;          // maybe_refresh, quant.cpp:303-311
    if (LITERAL && lit_step) {                           // detect_outliers verbatim, quant.cpp:313-335
        const double mx = block_max((active && !in) ? peak : 0.0, red);
        const bool trig = !(__ddiv_rn(mx, qa) <= kc.s_in[t]);
        if (trig && peak > kc.theta) in = true;
    } else if (peak > kc.theta) {                        // channel-local form (exact under C(t))
        in = true;
    }
    if (in) {                                            // fake_quant_step, quant.cpp:337-351
        const double os = scale_from_peak(peak, qo);
#pragma unroll
        for (int m = 0; m < N; ++m) x[m] = dmul(quant_code_div(x[m], os, qo), os);
    } else {
        const double S = kc.s_in[t], inv = __ddiv_rn(1.0, S);
#pragma unroll
        for (int m = 0; m < N; ++m) x[m] = dmul(quant_code_inv(x[m], S, inv, qa), S);
    }
    if (p.masks && active)
        p.masks[((static_cast<size_t>(kind) * p.S + s) * p.T + t) * p.E + i] = in ? 1 : 0;
}

// SpikeHook::spikes_at (quant.cpp:420-439): the step spikes with probability
// `rate` from a mix64 chain over (salt, sample, block, dir, t); the channels are
// the first min(channels, E) distinct picks of a further mix64 chain.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // quant.cpp:20-25
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ bool spike_hits(const SpikeCfg& sp, uint64_t sample, uint64_t t, uint64_t e, uint64_t ch) {
    uint64_t key = sp.salt;
    key = mix64(key ^ (0x5151ull + sample));
    key = mix64(key ^ (static_cast<uint64_t>(sp.block) * 131ull + static_cast<uint64_t>(sp.dir)));
    key = mix64(key ^ t);
    const double u = static_cast<double>(key >> 11) * 0x1.0p-53;
    if (u >= sp.rate) return false;
    uint64_t picks[kMaxSpikeChannels];
    const uint64_t want = min(static_cast<uint64_t>(sp.channels), e);
    uint64_t n = 0, pick = key;
    bool hit = false;
    while (n < want) {
        pick = mix64(pick);
        const uint64_t c = pick % e;
        bool dup = false;
        for (uint64_t j = 0; j < n; ++j) dup |= picks[j] == c;
        if (!dup) {
            picks[n++] = c;
            hit |= c == ch;
        }
    }
    return hit;
}

template <bool LITERAL, int N>
__global__ void __launch_bounds__(LITERAL ? 1024 : 128) k3_scan(const ScanParams p) {
    __shared__ double red[32];
    const int s = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = i < p.E;
    const int E = p.E, T = p.T, P = E + 2 * N;
    const double qa = qmax_for(p.abits), qo = qmax_for(p.obits);
    double A[N], h[N];
#pragma unroll
    for (int m = 0; m < N; ++m) {
        A[m] = active ? p.a[static_cast<size_t>(i) * N + m] : 0.0;
        h[m] = 0.0;
    }
    const double bd = active ? p.b_delta[i] : 0.0;
    bool inA = false, inB = false, inH = false;
    for (int t = 0; t < T; ++t) {
        const int c = row_at(p.order, t, T, p.grid);
        const double* pr = p.proj + (static_cast<size_t>(s) * T + t) * P;
        const double dpre = active ? pr[i] : 0.0;
        const double uv = active ? p.u[(static_cast<size_t>(s) * T + c) * E + i] : 0.0;
        const bool lit = LITERAL && (p.force_literal || (p.literal && p.literal[t]));
        const double delta = softplus_d(dadd(dpre, bd));  // ssm.cpp:150-151
        double a[N], b[N];
#pragma unroll
        for (int m = 0; m < N; ++m) {
            a[m] = gl::exp(dmul(delta, A[m]));
            b[m] = dmul(delta, __ldg(pr + E + m));
        }
        if (p.spike.rate > 0.0 && active &&
            spike_hits(p.spike, static_cast<uint64_t>(p.spike.sample0 + s), static_cast<uint64_t>(t),
                       static_cast<uint64_t>(E), static_cast<uint64_t>(i))) {
#pragma unroll
            for (int m = 0; m < N; ++m) b[m] = dmul(b[m], p.spike.gain);  // SpikeHook::on_inputs, before QuantHook
        }
        quant_row<LITERAL, N>(a, inA, 0, t, p, i, active, lit, qa, qo, red, s);
        quant_row<LITERAL, N>(b, inB, 1, t, p, i, active, lit, qa, qo, red, s);
#pragma unroll
        for (int m = 0; m < N; ++m) h[m] = dadd(dmul(a[m], h[m]), dmul(b[m], uv));
        quant_row<LITERAL, N>(h, inH, 2, t, p, i, active, lit, qa, qo, red, s);
        double o = 0.0;
#pragma unroll
        for (int m = 0; m < N; ++m) o = dadd(o, dmul(__ldg(pr + E + N + m), h[m]));
        if (active) p.o[(static_cast<size_t>(s) * T + c) * E + i] = o;
    }
}

cudaError_t launch_scan(const ScanParams& p, cudaStream_t st, bool* used_literal) {
    if (p.N != 16 || p.E < 1 || p.T < 1 || p.S < 1) return cudaErrorInvalidValue;
    if (p.spike.rate > 0.0 && (p.spike.channels < 1 || p.spike.channels > kMaxSpikeChannels)) return cudaErrorInvalidValue;
    bool lit = false;
    if (p.mode == MODE_DYNAMIC) {
        lit = p.force_literal != 0 || (p.literal != nullptr && p.literal_any != 0);
    }
    if (used_literal) *used_literal = lit;
    if (lit) {
        if (p.E > 1024) return cudaErrorInvalidValue;
        const int threads = ((p.E + 31) / 32) * 32;
        k3_scan<true, 16><<<dim3(1, p.S), threads, 0, st>>>(p);
        ++kernel_launch_counter();
    } else {
        const int threads = 128;
        k3_scan<false, 16><<<dim3((p.E + threads - 1) / threads, p.S), threads, 0, st>>>(p);
        ++kernel_launch_counter();
    }
    return cudaGetLastError();
}

}  // namespace ob
