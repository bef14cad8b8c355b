// K4 — auxiliary kernels of the Vim forward (< 1 % of the work): the f64
// projection GEMM used for patch embedding, the head and the FP (calibration /
// bypass) linear layers; patch gather; causal depthwise conv; mean pool.
// Each keeps the reference's per-output operation order so FP results match
// the CPU reference bit-for-bit (exp/log1p are glibc's, glibc_math.cuh).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace ob {

// Y[m][r] = 0.0 + sum_{k ascending} A[m][k] * W[r][k]  (detail::mm !ta,tb;
// tensor.cpp:373-382), 128x64 output tile per CTA, 8x4 per thread, k staged
// through shared memory 16 at a time, the next k tile loaded into registers
// while the current one is multiplied. Every output keeps its own sequential
// k order, so tiling does not change a bit of the result. FP64-bound: a MAC is a
// separately rounded DMUL + DADD (the reference builds with -ffp-contract=off).
// Small problems (fewer 128x64 tiles than SMs, e.g. the batch-1 patch embedding:
// 6 CTAs of 256 threads for 196 x 192 outputs, 104 us) take 16x16 tiles, one output
// per thread (TM = TN = 1): the same per-output k order, 156 CTAs.
constexpr int DG_BK = 16;

template <int TM, int TN>
__global__ void __launch_bounds__(256) k4_dgemm(const DGemmParams p) {
    constexpr int DG_BM = 16 * TM, DG_BN = 16 * TN, DG_TM = TM;
    __shared__ double sa[DG_BK][DG_BM + 1];
    __shared__ double sw[DG_BK][DG_BN + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * DG_BM, r0 = blockIdx.x * DG_BN;
    double acc[DG_TM][TN];
#pragma unroll
    for (int i = 0; i < DG_TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
    // k-tile element idx = threadIdx.x + 256 * u: row idx / 16, k idx % 16 (128 B runs)
    double ra[DG_BM * DG_BK / 256], rw[DG_BN * DG_BK / 256];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int u = 0; u < DG_BM * DG_BK / 256; ++u) {
            const int idx = threadIdx.x + 256 * u, r = idx / DG_BK, gk = k0 + idx % DG_BK, gm = m0 + r;
            ra[u] = (gm < p.M && gk < p.K) ? __ldg(p.a + static_cast<size_t>(gm) * p.lda + gk) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < DG_BN * DG_BK / 256; ++u) {
            const int idx = threadIdx.x + 256 * u, r = idx / DG_BK, gk = k0 + idx % DG_BK, gr = r0 + r;
            rw[u] = (gr < p.R && gk < p.K) ? __ldg(p.w + static_cast<size_t>(gr) * p.K + gk) : 0.0;
        }
    };
    fetch(0);
    for (int k0 = 0; k0 < p.K; k0 += DG_BK) {
#pragma unroll
        for (int u = 0; u < DG_BM * DG_BK / 256; ++u) {
            const int idx = threadIdx.x + 256 * u;
            sa[idx % DG_BK][idx / DG_BK] = ra[u];
        }
#pragma unroll
        for (int u = 0; u < DG_BN * DG_BK / 256; ++u) {
            const int idx = threadIdx.x + 256 * u;
            sw[idx % DG_BK][idx / DG_BK] = rw[u];
        }
        __syncthreads();
        if (k0 + DG_BK < p.K) fetch(k0 + DG_BK);  // in flight during this tile's products
        const int kk = min(DG_BK, p.K - k0);
        for (int k = 0; k < kk; ++k) {
            double av[DG_TM], wv[TN];
#pragma unroll
            for (int i = 0; i < DG_TM; ++i) av[i] = sa[k][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < TN; ++j) wv[j] = sw[k][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < DG_TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = dadd(acc[i][j], dmul(av[i], wv[j]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < DG_TM; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= p.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int r = r0 + tx + 16 * j;
            if (r >= p.R) continue;
            double y = dadd(0.0, acc[i][j]);
            const GemmEpi& e = p.epi;
            switch (e.post) {
                case POST_INPROJ:
                    if (r >= e.split) {
                        e.out2[static_cast<size_t>(m) * e.split + (r - e.split)] = y;  // SiLU applied by K1 (merge)
                        continue;
                    }
                    break;
                case POST_RESID: y = dadd(e.out[static_cast<size_t>(m) * e.ld_out + r], y); break;
                case POST_BIAS: y = dadd(y, e.bias[r]); break;
                case POST_XPROJ:
                    if (r < e.split) y = softplus_d(dadd(y, e.bias[r]));
                    break;
                default: break;
            }
            e.out[static_cast<size_t>(m) * e.ld_out + r] = y;
        }
    }
}

cudaError_t launch_dgemm(const DGemmParams& p, cudaStream_t st) {
    if (p.M < 1 || p.R < 1 || p.K < 1) return cudaErrorInvalidValue;
    const long big_tiles = static_cast<long>((p.R + 63) / 64) * ((p.M + 127) / 128);
    if (big_tiles >= 148) {
        k4_dgemm<8, 4><<<dim3((p.R + 63) / 64, (p.M + 127) / 128), 256, 0, st>>>(p);
    } else {
        k4_dgemm<1, 1><<<dim3((p.R + 15) / 16, (p.M + 15) / 16), 256, 0, st>>>(p);
    }
    ++kernel_launch_counter();
    return cudaGetLastError();
}

// patches[s][t][p] = img[s][gather(t,p)] with gather of ssm.cpp:72-84:
// (grid row, grid col, patch row, patch col, channel).
// One block per patch (sample, token): patch row pr is patch*channels contiguous
// doubles of image row gr*patch + pr, so reads and writes are coalesced and the
// index arithmetic is 32-bit within the patch.
__global__ void __launch_bounds__(256) k4_patch_gather(const double* __restrict__ img, double* __restrict__ patches,
                                                       int S, int image, int channels, int patch) {
    const int g = image / patch, L = g * g, rowv = patch * channels, pv = patch * rowv;
    const size_t st = blockIdx.x;  // sample * L + token
    const int t = static_cast<int>(st % L);
    const size_t s = st / L;
    const int gr = t / g, gc = t % g;
    const double* src = img + s * static_cast<size_t>(image) * image * channels +
                        (static_cast<size_t>(gr * patch) * image + gc * patch) * channels;
    double* dst = patches + st * pv;
    for (int j = threadIdx.x; j < pv; j += blockDim.x) {
        const int pr = j / rowv, off = j - pr * rowv;
        dst[j] = __ldg(src + static_cast<size_t>(pr) * image * channels + off);
    }
}

cudaError_t launch_patch_gather(const double* img, double* patches, int S, int image, int channels, int patch,
                                cudaStream_t st) {
    const int g = image / patch;
    const unsigned blocks = static_cast<unsigned>(S) * static_cast<unsigned>(g * g);
    if (blocks == 0) return cudaSuccess;
    k4_patch_gather<<<blocks, 256, 0, st>>>(img, patches, S, image, channels, patch);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

// Depthwise causal conv over tokens, ssm.cpp:200-212:
// u[t][c] = 0.0 + sum_{k ascending, t-(W-1-k) >= 0} taps[c][k] * u0[t-(W-1-k)][c].
__global__ void k4_conv(const double* __restrict__ u0, const double* __restrict__ taps, double* __restrict__ u,
                        int S, int T, int E, int W) {
    const size_t total = static_cast<size_t>(S) * T * E;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % E);
        const int t = static_cast<int>((i / E) % T);
        const size_t base = i - static_cast<size_t>(t) * E;  // (s, 0, c)
        double s = 0.0;
        for (int k = 0; k < W; ++k) {
            const int src = t - (W - 1 - k);
            if (src < 0) continue;
            s = dadd(s, dmul(taps[c * W + k], u0[base + static_cast<size_t>(src) * E]));
        }
        u[i] = s;
    }
}

// Fast form for W = 4 and even E: a thread owns two channels of a run of kRun
// tokens; the run's inputs (plus W-1 halo tokens) are loaded once, as 16-byte
// vectors, before any output is formed. Same per-output order as k4_conv.
template <int W>
__global__ void __launch_bounds__(128) k4_conv_run(const double* __restrict__ u0, const double* __restrict__ taps,
                                                   double* __restrict__ u, int S, int T, int E) {
    constexpr int kRun = 14;
    const int ch = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (ch >= E) return;
    const int nrun = (T + kRun - 1) / kRun;
    const int s = blockIdx.y / nrun, t0 = (blockIdx.y % nrun) * kRun, t1 = min(T, t0 + kRun);
    double2 tp[W];
#pragma unroll
    for (int k = 0; k < W; ++k) tp[k] = make_double2(__ldg(taps + ch * W + k), __ldg(taps + (ch + 1) * W + k));
    const double* base = u0 + static_cast<size_t>(s) * T * E + ch;
    double2 in[kRun + W - 1];  // in[j] = token t0 - (W-1) + j
#pragma unroll
    for (int j = 0; j < kRun + W - 1; ++j) {
        const int tok = t0 - (W - 1) + j;
        in[j] = (tok >= 0 && tok < t1) ? __ldg(reinterpret_cast<const double2*>(base + static_cast<size_t>(tok) * E))
                                       : make_double2(0.0, 0.0);
    }
    double* out = u + static_cast<size_t>(s) * T * E + ch;
#pragma unroll
    for (int i = 0; i < kRun; ++i) {
        const int t = t0 + i;
        if (t >= t1) break;
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            if (t - (W - 1 - k) < 0) continue;  // ssm.cpp:200-212 skips taps before the sequence start
            a = dadd(a, dmul(tp[k].x, in[i + k].x));
            b = dadd(b, dmul(tp[k].y, in[i + k].y));
        }
        *reinterpret_cast<double2*>(out + static_cast<size_t>(t) * E) = make_double2(a, b);
    }
}

cudaError_t launch_conv(const double* u0, const double* taps, double* u, int S, int T, int E, int W, cudaStream_t st) {
    if (W == 4 && E % 2 == 0 && (reinterpret_cast<uintptr_t>(u0) & 15) == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0) {
        const int nrun = (T + 13) / 14;
        dim3 grid((E / 2 + 127) / 128, S * nrun);
        k4_conv_run<4><<<grid, 128, 0, st>>>(u0, taps, u, S, T, E);
        ++kernel_launch_counter();
    } else {
        k4_conv<<<2368, 256, 0, st>>>(u0, taps, u, S, T, E, W);
        ++kernel_launch_counter();
    }
    return cudaGetLastError();
}

// pooled[s][i] = (sum_{t ascending} x[s][t][i]) * (1/T), ssm.cpp:266-270.
__global__ void k4_meanpool(const double* __restrict__ x, double* __restrict__ pooled, int S, int T, int E) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (i >= E) return;
    double acc = 0.0;
    const double* xs = x + static_cast<size_t>(s) * T * E + i;
    int t = 0;
    for (; t + 8 <= T; t += 8) {  // eight rows' loads in flight, then the sums in ascending t
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = xs[static_cast<size_t>(t + j) * E];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = dadd(acc, v[j]);
    }
    for (; t < T; ++t) acc = dadd(acc, xs[static_cast<size_t>(t) * E]);
    pooled[static_cast<size_t>(s) * E + i] = dmul(acc, __ddiv_rn(1.0, static_cast<double>(T)));
}

cudaError_t launch_meanpool(const double* x, double* pooled, int S, int T, int E, cudaStream_t st) {
    k4_meanpool<<<dim3((E + 127) / 128, S), 128, 0, st>>>(x, pooled, S, T, E);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

// The device transcendental functions of the path (glibc's exp / log1p and the
// softplus / SiLU built on them, common.cuh) over a vector, for the tests that pin
// them to the reference's libm.
__global__ void k4_math_eval(int fn, const double* __restrict__ x, double* __restrict__ y, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double v = x[i];
        y[i] = fn == 0 ? gl::exp(v) : fn == 1 ? gl::log1p(v) : fn == 2 ? softplus_d(v) : silu_d(v);
    }
}
cudaError_t launch_math_eval(int fn, const double* x, double* y, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 16));
    k4_math_eval<<<blocks, 256, 0, st>>>(fn, x, y, n);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

// FP64 pipe probe: 8 independent DFMA chains per thread, 4 CTAs x 256 threads
// per SM; the result is folded into a store so nothing is dead code.
__global__ void __launch_bounds__(256) k4_dfma_probe(double* out, int iters, double a, double b) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = fma(v[j], a, b);
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
    if (s == 12345.678) out[0] = s;
}

double measure_fp64_peak(cudaStream_t st, int num_sms) {
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 0.0;
    const int iters = 4096, blocks = num_sms * 4, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k4_dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, st);
        k4_dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    return flops / (best * 1e-3) / 1e12;
}

}  // namespace ob
