// K1 over streams of K x C planes, and the GPU-backed gemm-bench stage
// (bench_gemm, bench_refresh_sweep: gemm.cpp:260-411).
//
// The reference's detect_outliers takes a plane of E channels x n values
// (quant.cpp:313-335): a channel's peak is its max |x| over the n values, the
// scan fires when max_{ch not in O} peak / q_a exceeds S^I(t), and then adds
// every channel whose peak exceeds theta. split_quantize (gemm.cpp:106-135)
// codes inlier values at S^I(t) and each outlier channel at its own scale
// peak / q_o. Only the outlier list is sequential in t, so:
//   kp_peaks     every (step, channel) peak at once (warp per channel row);
//   kp_walk      one warp walks the steps: refresh, detect, per-step mask words,
//                |O(t)| and DetectResult::scanned (the only serial part);
//   kp_quantize  every plane in parallel into the QAct operand of K2, row
//                r = t*C + i (the reference's y[m][c] is K2's out[r][m]);
// and K2 runs all steps' GEMMs as one launch (each row's output depends only
// on its own row, so this equals the reference's per-step hybrid_gemm).
#include <algorithm>
#include <cuda_fp16.h>
#include <vector>

#include "common.cuh"
#include "engine.h"
#include "kernels.h"
#include "planes.h"
#include "seeded_rng.h"

namespace ob {

constexpr int kMaxPlaneWords = 128;  // K <= 4096 channels per plane

// peaks[row] = max(0, max_i |x[row][i]|) with NaN ignored (std::max fold, quant.cpp:318-320)
__global__ void __launch_bounds__(256) kp_peaks(const double* __restrict__ x, double* __restrict__ peaks, long rows,
                                                int C) {
    const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const double* xr = x + r * C;
    double m = 0.0;
    for (int i = lane; i < C; i += 32) m = fmax(m, fabs(xr[i]));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) peaks[r] = m;
}

// maybe_refresh + detect_outliers over the steps (quant.cpp:303-335). Lane l
// owns channels 32w + l; bit w of `in` = channel 32w + l is in O.
__global__ void __launch_bounds__(32) kp_walk(const double* __restrict__ peaks, const double* __restrict__ s_in,
                                              int steps, int K, double theta, double qa, int n_refresh,
                                              uint32_t* __restrict__ omask_t, int* __restrict__ count,
                                              uint8_t* __restrict__ scanned) {
    const int lane = threadIdx.x;
    const int J = (K + 31) / 32;
    unsigned long long in[kMaxPlaneWords / 64] = {0ull, 0ull};
    for (int t = 0; t < steps; ++t) {
        if (n_refresh != 0 && t != 0 && t % n_refresh == 0) in[0] = in[1] = 0ull;
        const double* pk = peaks + static_cast<size_t>(t) * K;
        double mx = 0.0;
        for (int w = 0; w < J; ++w) {
            const int ch = 32 * w + lane;
            if (ch < K && !((in[w >> 6] >> (w & 63)) & 1ull)) mx = fmax(mx, pk[ch]);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double s_dyn = __ddiv_rn(mx, qa);
        const bool scan = !(s_dyn <= s_in[t]);  // quant.cpp:322: returns unless s_dyn > S^I
        int cnt = 0;
        for (int w = 0; w < J; ++w) {
            const int ch = 32 * w + lane;
            if (scan && ch < K && pk[ch] > theta) in[w >> 6] |= 1ull << (w & 63);
            const unsigned word = __ballot_sync(0xffffffffu, ch < K && ((in[w >> 6] >> (w & 63)) & 1ull));
            if (lane == 0) omask_t[static_cast<size_t>(t) * J + w] = word;
            cnt += __popc(word);
        }
        if (lane == 0) {
            count[t] = cnt;
            if (scanned) scanned[t] = scan ? 1 : 0;
        }
    }
}

// split_quantize of every plane (gemm.cpp:106-135) into QAct rows r = t*C + i.
// Block: 32 channels x 32 values of one step, transposed through shared memory.
__global__ void __launch_bounds__(256) kp_quantize(const double* __restrict__ x, const double* __restrict__ peaks,
                                                   const double* __restrict__ s_in,
                                                   const uint32_t* __restrict__ omask_t, const int* __restrict__ count,
                                                   int K, int Kp, int C, double qa, double qo, QAct a) {
    __shared__ double tile[32][33];
    const int t = blockIdx.z, ch0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int J = (K + 31) / 32;
    for (int r = ty; r < 32; r += 8) {  // tile[ch][i] = x[t][ch0 + r][i0 + tx]
        const int ch = ch0 + r, i = i0 + tx;
        tile[r][tx] = (ch < K && i < C) ? x[(static_cast<size_t>(t) * K + ch) * C + i] : 0.0;
    }
    __syncthreads();
    const int ch = ch0 + tx;
    const double S = s_in[t];
    const bool o = ch < K && ((omask_t[static_cast<size_t>(t) * J + (ch >> 5)] >> (ch & 31)) & 1u);
    const double os = o ? scale_from_peak(peaks[static_cast<size_t>(t) * K + ch], qo) : 0.0;
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r;
        if (i >= C || ch >= Kp) continue;
        const size_t row = static_cast<size_t>(t) * C + i;
        const double v = tile[tx][r];
        int8_t code = 0;
        if (ch < K) {
            if (o) {
                a.ocode[row * Kp + ch] = static_cast<int8_t>(static_cast<int>(quant_code_div(v, os, qo)));
                a.oscale[row * Kp + ch] = os;
            } else {
                code = static_cast<int8_t>(static_cast<int>(quant_code_div(v, S, qa)));
            }
        }
        a.codes[row * Kp + ch] = code;
        if (blockIdx.x == 0 && tx < a.J) {  // row metadata: mask words (0 beyond K), |O(t)|, S^I(t)
            for (int w = tx; w < a.J; w += 32) a.omask[row * a.J + w] = w < J ? omask_t[static_cast<size_t>(t) * J + w] : 0u;
            if (tx == 0) {
                a.ocnt[row] = count[t];
                a.s_row[row] = S;
            }
        }
    }
}

size_t plane_workspace_bytes(int steps, int K) {
    const size_t J = (K + 31) / 32;
    return static_cast<size_t>(steps) * K * sizeof(double) + static_cast<size_t>(steps) * J * sizeof(uint32_t) +
           static_cast<size_t>(steps) * sizeof(int) + 64;
}

cudaError_t launch_detect_planes(const PlaneParams& p, cudaStream_t st) {
    if (p.steps < 1 || p.K < 1 || p.K > 32 * kMaxPlaneWords || p.C < 1 || p.Kp < p.K || p.a.J < (p.Kp + 31) / 32 ||
        !p.work)
        return cudaErrorInvalidValue;
    const int J = (p.K + 31) / 32;
    double* peaks = static_cast<double*>(p.work);
    uint32_t* omask_t = reinterpret_cast<uint32_t*>(peaks + static_cast<size_t>(p.steps) * p.K);
    int* count = reinterpret_cast<int*>(omask_t + static_cast<size_t>(p.steps) * J);
    const long rows = static_cast<long>(p.steps) * p.K;
    kp_peaks<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(p.x, peaks, rows, p.C);
    kp_walk<<<1, 32, 0, st>>>(peaks, p.s_in, p.steps, p.K, p.theta, qmax_for(p.abits), p.n_refresh, omask_t, count,
                              p.scanned);
    dim3 grid((p.Kp + 31) / 32, (p.C + 31) / 32, p.steps);
    kp_quantize<<<grid, 256, 0, st>>>(p.x, peaks, p.s_in, omask_t, count, p.K, p.Kp, p.C, qmax_for(p.abits),
                                      qmax_for(p.obits), p.a);
    kernel_launch_counter() += 3;
    if (p.count_out) {
        const cudaError_t e = cudaMemcpyAsync(p.count_out, count, static_cast<size_t>(p.steps) * sizeof(int),
                                              cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

// f16_output: every output value through IEEE binary16, round to nearest even
// (round_f16, gemm.cpp:245-258)
__global__ void kp_round_f16(double* y, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        y[i] = static_cast<double>(__half2float(__double2half(y[i])));
}

namespace {

template <class T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    Dev(const std::vector<T>& v, cudaStream_t st) : Dev(v.size()) {
        cuda_check(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
    }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

double median_of(std::vector<double> v) {  // gemm.cpp:40-44
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair() {
        cuda_check(cudaEventCreate(&a), "event");
        cuda_check(cudaEventCreate(&b), "event");
    }
    ~EventPair() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    double ns() const {
        float ms = 0.0f;
        cuda_check(cudaEventElapsedTime(&ms, a, b), "event time");
        return static_cast<double>(ms) * 1e6;
    }
};

// Weight plane of K2 from codes [m][k]: K-major [Rp][Kp] and its transpose.
void weight_planes(const std::vector<int8_t>& wc, size_t m, size_t k, size_t Rp, size_t Kp, std::vector<int8_t>& w,
                   std::vector<int8_t>& wt) {
    w.assign(Rp * Kp, 0);
    wt.assign(Kp * Rp, 0);
    for (size_t r = 0; r < m; ++r)
        for (size_t c = 0; c < k; ++c) wt[c * Rp + r] = w[r * Kp + c] = wc[r * k + c];
}

}  // namespace

std::vector<SweepRecord> refresh_sweep(const SweepSettings& s, cudaStream_t st, int num_sms,
                                       std::vector<double>* outputs) {
    // validation and data generation: bench_refresh_sweep (gemm.cpp:326-372), same draws
    require(!s.periods.empty(), "refresh sweep: need at least one period");
    require(s.steps >= 2 && s.trials >= 1, "refresh sweep: need steps >= 2 and trials >= 1");
    require(s.persistent_channels <= s.k, "refresh sweep: more persistent channels than channels");
    require(s.transient_rate >= 0.0 && s.transient_rate <= 1.0, "refresh sweep: transient rate must be in [0, 1]");
    require(s.spike_gain > 1.0, "refresh sweep: spike gain must exceed 1");
    require(s.k >= 1 && s.k <= 32 * static_cast<size_t>(kMaxPlaneWords), "refresh sweep: k out of range (1..4096)");
    require(s.m >= 1 && s.c >= 1, "refresh sweep: m and c must be positive");
    SeededRng rng(s.seed);
    const size_t steps = s.steps, k = s.k, c = s.c, m = s.m;
    std::vector<double> clean(steps * k * c);
    rng.fill_normal(clean, 0.0, 1.0);
    std::vector<size_t> all(k);
    for (size_t i = 0; i < k; ++i) all[i] = i;
    for (size_t i = 0; i < s.persistent_channels; ++i) std::swap(all[i], all[i + rng.below(k - i)]);
    const std::vector<size_t> persistent(all.begin(), all.begin() + static_cast<std::ptrdiff_t>(s.persistent_channels));
    std::vector<double> spiked = clean;
    for (size_t t = 0; t < steps; ++t) {
        double* plane = spiked.data() + t * k * c;
        for (size_t ch : persistent)
            for (size_t i = 0; i < c; ++i) plane[ch * c + i] *= s.spike_gain;
        if (rng.uniform() < s.transient_rate) {
            const size_t ch = rng.below(k);
            for (size_t i = 0; i < c; ++i) plane[ch * c + i] *= s.spike_gain;
        }
    }
    const double qmax = 7.0;
    std::vector<double> scale_inlier(steps);
    double theta = 0.0;
    for (size_t t = 0; t < steps; ++t) {
        double mx = 0.0;
        const double* plane = clean.data() + t * k * c;
        for (size_t i = 0; i < k * c; ++i) mx = std::max(mx, std::fabs(plane[i]));
        scale_inlier[t] = mx == 0.0 ? 1.0 : mx / qmax;
        theta = std::max(theta, mx);
    }
    theta *= 1.05;
    std::vector<int8_t> wc(m * k);
    for (auto& v : wc) v = static_cast<int8_t>(static_cast<int>(rng.below(15)) - 7);
    std::vector<double> w_scales(m);
    for (auto& v : w_scales) v = rng.uniform(0.005, 0.02);

    // device operands
    const size_t Kp = round_up(k, 16), Rp = round_up(m, 32), J = (Kp + 31) / 32, rows = steps * c;
    std::vector<int8_t> w, wt;
    weight_planes(wc, m, k, Rp, Kp, w, wt);
    std::vector<double> ws(Rp, 0.0);
    std::copy(w_scales.begin(), w_scales.end(), ws.begin());
    Dev<double> dx(spiked, st), dsin(scale_inlier, st), dws(ws, st), dy(rows * Rp);
    Dev<int8_t> dw(w, st), dwt(wt, st), codes(rows * Kp), ocode(rows * Kp);
    Dev<double> oscale(rows * Kp), s_row(rows);
    Dev<int> ocnt(rows), count(steps);
    Dev<uint32_t> omask(rows * J);
    Dev<uint8_t> scanned(steps);
    Dev<unsigned char> work(plane_workspace_bytes(static_cast<int>(steps), static_cast<int>(k)));
    PlaneParams pp;
    pp.x = dx.p;
    pp.steps = static_cast<int>(steps);
    pp.K = static_cast<int>(k);
    pp.Kp = static_cast<int>(Kp);
    pp.C = static_cast<int>(c);
    pp.theta = theta;
    pp.s_in = dsin.p;
    pp.abits = 4;
    pp.obits = 8;
    pp.a = QAct{codes.p, nullptr, s_row.p, ocnt.p, omask.p, ocode.p, oscale.p, static_cast<int>(J)};
    pp.scanned = scanned.p;
    pp.work = work.p;
    pp.count_out = count.p;
    QLinParams q;
    q.M = static_cast<int>(rows);
    q.R = static_cast<int>(Rp);
    q.K = static_cast<int>(Kp);
    q.a = pp.a;
    q.w = dw.p;
    q.wt = dwt.p;
    q.ws = dws.p;
    q.epi.post = POST_STORE;
    q.epi.out = dy.p;
    q.epi.ld_out = static_cast<int>(Rp);

    std::vector<SweepRecord> out;
    if (outputs) outputs->clear();
    EventPair ev;
    for (size_t period : s.periods) {
        pp.n_refresh = static_cast<int>(period);
        std::vector<double> totals(s.trials);
        for (size_t trial = 0; trial < s.trials; ++trial) {
            cuda_check(cudaEventRecord(ev.a, st), "event");
            cuda_check(launch_detect_planes(pp, st), "detect planes");
            cuda_check(launch_qlinear(q, st, num_sms), "quant linear");
            cuda_check(cudaEventRecord(ev.b, st), "event");
            cuda_check(cudaEventSynchronize(ev.b), "event sync");
            totals[trial] = ev.ns();
        }
        std::vector<int> cnt(steps);
        std::vector<uint8_t> sc(steps);
        cuda_check(cudaMemcpyAsync(cnt.data(), count.p, steps * sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaMemcpyAsync(sc.data(), scanned.p, steps, cudaMemcpyDeviceToHost, st), "D2H");
        if (outputs) {
            std::vector<double> y(rows * Rp);
            cuda_check(cudaMemcpyAsync(y.data(), dy.p, y.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
            cuda_check(cudaStreamSynchronize(st), "sync");
            for (size_t r = 0; r < rows; ++r)  // [step][column][m]
                outputs->insert(outputs->end(), y.begin() + static_cast<std::ptrdiff_t>(r * Rp),
                                y.begin() + static_cast<std::ptrdiff_t>(r * Rp + m));
        }
        cuda_check(cudaStreamSynchronize(st), "sync");
        double o_accum = 0.0;
        size_t scans = 0;
        for (size_t t = 0; t < steps; ++t) {
            o_accum += static_cast<double>(cnt[t]);
            scans += sc[t];
        }
        SweepRecord rec;
        rec.period = period;
        rec.median_total_ns = median_of(totals);
        rec.mean_o_list = o_accum / static_cast<double>(steps);
        rec.scans_per_step = static_cast<double>(scans) / static_cast<double>(steps);
        out.push_back(rec);
    }
    return out;
}

std::vector<BenchRecord> gemm_bench(const BenchSettings& s, cudaStream_t st, int num_sms) {
    // bench_gemm (gemm.cpp:260-324): same validation, draws and operands; the
    // "hybrid" path is K2 on the split problem, "f64" the f64 GEMM of the
    // dequantized copies. Device time per trial (CUDA events), median.
    require(!s.sizes.empty(), "bench_gemm: need at least one size");
    require(s.trials >= 1, "bench_gemm: trials must be >= 1");
    require(s.outlier_fraction >= 0.0 && s.outlier_fraction <= 1.0, "bench_gemm: outlier fraction must be in [0, 1]");
    SeededRng rng(s.seed);
    std::vector<BenchRecord> out;
    EventPair ev;
    for (size_t n : s.sizes) {
        require(n >= 1 && n <= 43826196u, "bench_gemm: size out of range");
        size_t n_o = static_cast<size_t>(std::llround(s.outlier_fraction * static_cast<double>(n)));
        n_o = std::min(n_o, n);
        std::vector<int8_t> wc(n * n), xc(n * n);
        for (auto& v : wc) v = static_cast<int8_t>(static_cast<int>(rng.below(15)) - 7);
        for (auto& v : xc) v = static_cast<int8_t>(static_cast<int>(rng.below(15)) - 7);
        std::vector<double> w_scales(n);
        for (auto& v : w_scales) v = rng.uniform(0.005, 0.02);
        const double inl_scale = rng.uniform(0.005, 0.02);
        std::vector<size_t> all(n);
        for (size_t i = 0; i < n; ++i) all[i] = i;
        for (size_t i = 0; i < n_o; ++i) std::swap(all[i], all[i + rng.below(n - i)]);
        std::vector<size_t> o_list(all.begin(), all.begin() + static_cast<std::ptrdiff_t>(n_o));
        std::sort(o_list.begin(), o_list.end());
        std::vector<double> o_scales(n_o);
        for (auto& v : o_scales) v = rng.uniform(0.005, 0.02);
        std::vector<int8_t> plane = xc, ocodes(n_o * n);  // extract_outliers (gemm.cpp:84-104)
        for (size_t j = 0; j < n_o; ++j) std::fill(plane.begin() + o_list[j] * n, plane.begin() + (o_list[j] + 1) * n, 0);
        for (auto& v : ocodes) v = static_cast<int8_t>(static_cast<int>(rng.below(255)) - 127);

        // K2 operands: rows = the plane's columns (tokens), channels = its rows
        const size_t Kp = round_up(n, 16), Rp = round_up(n, 32), Mp = n, J = (Kp + 31) / 32;
        std::vector<int8_t> w, wt, codes(Mp * Kp, 0), oc(Mp * Kp, 0);
        weight_planes(wc, n, n, Rp, Kp, w, wt);
        std::vector<double> ws(Rp, 0.0), os(Mp * Kp, 0.0), srow(Mp, inl_scale);
        std::copy(w_scales.begin(), w_scales.end(), ws.begin());
        std::vector<uint32_t> words(J, 0u), omask(Mp * J);
        for (size_t ch : o_list) words[ch / 32] |= 1u << (ch % 32);
        for (size_t r = 0; r < Mp; ++r) std::copy(words.begin(), words.end(), omask.begin() + r * J);
        for (size_t kk = 0; kk < n; ++kk)
            for (size_t col = 0; col < n; ++col) codes[col * Kp + kk] = plane[kk * n + col];
        for (size_t j = 0; j < n_o; ++j)
            for (size_t col = 0; col < n; ++col) {
                oc[col * Kp + o_list[j]] = ocodes[j * n + col];
                os[col * Kp + o_list[j]] = o_scales[j];
            }
        std::vector<int> ocnt(Mp, static_cast<int>(n_o));
        // f64 reference operands (dequantized copies), B transposed for the K-major f64 GEMM
        std::vector<double> a(n * n), bt(n * n);
        for (size_t r = 0; r < n; ++r)
            for (size_t col = 0; col < n; ++col) a[r * n + col] = w_scales[r] * wc[r * n + col];
        for (size_t r = 0; r < n; ++r)
            for (size_t col = 0; col < n; ++col) bt[col * n + r] = inl_scale * plane[r * n + col];
        for (size_t j = 0; j < n_o; ++j)
            for (size_t col = 0; col < n; ++col) bt[col * n + o_list[j]] = o_scales[j] * ocodes[j * n + col];

        Dev<int8_t> dw(w, st), dwt(wt, st), dcodes(codes, st), doc(oc, st);
        Dev<double> dws(ws, st), dos(os, st), dsrow(srow, st), dy(Mp * Rp), da(a, st), dbt(bt, st), dyf(n * n);
        Dev<int> docnt(ocnt, st);
        Dev<uint32_t> domask(omask, st);
        QLinParams q;
        q.M = static_cast<int>(Mp);
        q.R = static_cast<int>(Rp);
        q.K = static_cast<int>(Kp);
        q.a = QAct{dcodes.p, nullptr, dsrow.p, docnt.p, domask.p, doc.p, dos.p, static_cast<int>(J)};
        q.w = dw.p;
        q.wt = dwt.p;
        q.ws = dws.p;
        q.epi.post = POST_STORE;
        q.epi.out = dy.p;
        q.epi.ld_out = static_cast<int>(Rp);
        DGemmParams g;
        g.M = static_cast<int>(n);
        g.R = static_cast<int>(n);
        g.K = static_cast<int>(n);
        g.a = da.p;
        g.lda = static_cast<int>(n);
        g.w = dbt.p;
        g.epi.post = POST_STORE;
        g.epi.out = dyf.p;
        g.epi.ld_out = static_cast<int>(n);
        std::vector<double> th(s.trials), tf(s.trials);
        for (size_t t = 0; t < s.trials; ++t) {
            cuda_check(cudaEventRecord(ev.a, st), "event");
            cuda_check(launch_qlinear(q, st, num_sms), "quant linear");
            if (s.f16_output) {
                kp_round_f16<<<static_cast<unsigned>(std::min<size_t>((Mp * Rp + 255) / 256, 4096)), 256, 0, st>>>(
                    dy.p, Mp * Rp);
                ++kernel_launch_counter();
            }
            cuda_check(cudaEventRecord(ev.b, st), "event");
            cuda_check(cudaEventSynchronize(ev.b), "event sync");
            th[t] = ev.ns();
        }
        for (size_t t = 0; t < s.trials; ++t) {
            cuda_check(cudaEventRecord(ev.a, st), "event");
            cuda_check(launch_dgemm(g, st), "f64 gemm");
            cuda_check(cudaEventRecord(ev.b, st), "event");
            cuda_check(cudaEventSynchronize(ev.b), "event sync");
            tf[t] = ev.ns();
        }
        out.push_back({"hybrid", n, median_of(th)});
        out.push_back({"f64", n, median_of(tf)});
    }
    return out;
}

}  // namespace ob
