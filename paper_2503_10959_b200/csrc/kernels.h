// Kernel parameter blocks and launchers (host/device shared, internal to the
// library; the public boundary is include/ouro_b200.h).
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ob {

// Kernels launched by the calling host thread (every launch_* wrapper counts its
// <<<>>> launches; the engine reports per-op deltas as gpu_launches).
inline long& kernel_launch_counter() {
    static thread_local long n = 0;
    return n;
}

// Allow a kernel the device's opt-in shared-memory maximum (less its static
// shared memory), once per (kernel, device): the attribute caps what launches
// may request (so it is set to the device limit, not to one launch's size) and
// is per device (contexts on several devices may share a process).
template <auto Kernel>
cudaError_t ensure_smem_attr(int bytes) {
    static std::atomic<unsigned long long> done{0};  // bit d: set on device d
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa{};  // static + dynamic shared memory must fit the opt-in limit
    e = cudaFuncGetAttributes(&fa, Kernel);
    if (e != cudaSuccess) return e;
    const int limit = optin - static_cast<int>(fa.sharedSizeBytes);
    if (bytes > limit) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, limit);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

enum Mode { MODE_FP = 0, MODE_DYNAMIC = 1, MODE_STATIC = 2 };  // quant.hpp:101 (FP == bypass)
enum K1Src { K1_SRC_PLAIN = 0, K1_SRC_RMSNORM = 1, K1_SRC_MERGE = 2 };

// Calibration of one activation tensor (TensorCalib, quant.hpp:36-42), device side.
struct SiteCal {
    double theta = 0.0;
    const double* s_in = nullptr;    // [T]
    const double* s_full = nullptr;  // [T]
};

// Quantized activation operand of one quant-linear call: row m = (sample, step).
struct QAct {
    int8_t* codes = nullptr;      // [M][E] inlier codes, 0 at outlier positions
    uint8_t* codes4 = nullptr;    // or the same codes nibble-packed (A4): [M][E/2], low nibble = even channel
                                  // (pack_int4's layout, gemm.cpp:60-73, with the channels as its columns)
    double* s_row = nullptr;      // [M] inlier scale of the row's plane (S^I(t) or S_full(t))
    int* ocnt = nullptr;          // [M] |O(t)|
    uint32_t* omask = nullptr;    // [M][J] bit ch%32 of word ch/32: channel in O(t)
    int8_t* ocode = nullptr;      // [M][E] outlier codes (o_bits), valid at outlier positions only
    double* oscale = nullptr;     // [M][E] per-channel outlier scales, valid at outlier positions only
    int J = 0;                    // mask words per row, ceil(E/32)
};

struct K1Params {
    int S = 0, T = 0, E = 0;      // sequences (samples), steps, channels
    int src = K1_SRC_PLAIN;
    const double* x = nullptr;    // [S][T][E] canonical rows (PLAIN/RMSNORM) or o_dir0 (MERGE)
    const double* x2 = nullptr;   // o_dir1 (MERGE), may be null
    const double* gate = nullptr; // (MERGE)
    int order = -1, grid = 0;     // step t reads canonical row scan_perm(order, t); -1 = identity
    int mode = MODE_DYNAMIC, n_refresh = 10, abits = 8, obits = 8, window = 10;
    SiteCal cal;
    const double* inv_in = nullptr;    // optional [T] 1/s_in (host-computed); else divided in-kernel
    const double* inv_full = nullptr;  // optional [T] 1/s_full
    int force_literal = 0;             // run the literal detector kernel
    int window_kernel = 0;             // plain / RMSNorm channel-parallel path: 1 = the register window
                                       // kernel where E % 64 == 0, E <= 768 (A/B aid), 0 = the staged kernel
    // quantized outputs (rows in step order, row = s*T + t): the QAct operand
    int8_t* codes = nullptr;
    uint8_t* codes4 = nullptr;    // A4: the inlier codes nibble-packed instead (QAct::codes4), codes unused
    double* s_row = nullptr;
    int* ocnt = nullptr;
    uint32_t* omask = nullptr;    // [S*T][ceil(E/32)]
    int8_t* ocode = nullptr;      // [S*T][E] dense
    double* oscale = nullptr;     // [S*T][E] dense
    uint8_t* scanned = nullptr;   // optional [S*T] (DetectResult::scanned; literal kernel only)
    // FP mode outputs
    double* xout = nullptr;                 // [S*T][E] materialized input rows
    unsigned long long* peaks = nullptr;    // [T][E] running max |x| (f64 bits), calibration
};
cudaError_t launch_k1(const K1Params& p, cudaStream_t st);
// Several scan directions' K1 over the same rows: one launch on the staged fast
// path (each direction's outputs in its own QAct), else one launch each.
cudaError_t launch_k1_dirs(const K1Params* ps, int n, cudaStream_t st);

// Post-ops fused into the quant-linear / f64 GEMM epilogues.
enum PostOp {
    POST_STORE = 0,    // out[m][r] = y
    POST_INPROJ = 1,   // r <  E: u0[m][r] = y ; r >= E: gate_pre[m][r-E] = y (SiLU in the merge K1) (ssm.cpp:196-198)
    POST_RESID = 2,    // out[m][r] += y   (D1 residual)
    POST_BIAS = 3,     // out[m][r] = y + bias[r]  (patch embed / head, ssm.cpp:254-256, 271-274)
    POST_XPROJ = 4,    // r < split: out = softplus(y + bias[r]) (delta, ssm.cpp:150-151); else out = y (B | C)
};

struct GemmEpi {
    int post = POST_STORE;
    double* out = nullptr;        // [M][ld_out]
    int ld_out = 0;
    double* out2 = nullptr;       // gate for POST_INPROJ, [M][E]
    int split = 0;                // E for POST_INPROJ
    const double* bias = nullptr; // POST_BIAS
    int32_t* acc_in = nullptr;    // optional [M][R] (parity)
    int32_t* acc_out = nullptr;   // optional [M][R] (parity)
};

// K2: hybrid quant-linear, Y[m][r] = ws[r]*(S_m*acc[m][r] + sum_j (s_j*w[r][ch_j])*xo_j)
// (gemm.cpp:181-225) with the int8 inlier GEMM on tcgen05 kind::i8.
struct QLinParams {
    int M = 0, R = 0, K = 0;
    QAct a;                        // activation codes, row-major [M][K]
    const int8_t* w = nullptr;     // [R][K] weight codes (K-major), |code| <= 7
    const int8_t* wt = nullptr;    // [K][R] transposed codes for the outlier gather
    const double* ws = nullptr;    // [R] weight row scales
    GemmEpi epi;
};
cudaError_t launch_qlinear(const QLinParams& p, cudaStream_t st, int num_sms);

// f64 GEMM with the reference's per-output k-ascending sum (detail::mm,
// tensor.cpp:373-382): Y[m][r] = 0.0 + sum_k A[m][k] * W[r][k].
struct DGemmParams {
    int M = 0, R = 0, K = 0;
    const double* a = nullptr;   // [M][lda]
    int lda = 0;
    const double* w = nullptr;   // [R][K]
    GemmEpi epi;
};
cudaError_t launch_dgemm(const DGemmParams& p, cudaStream_t st);

// K3: selective scan with the QuantHook policy.
struct ScanKindCal {
    double theta = 0.0;
    const double* s_in = nullptr;
    const double* s_full = nullptr;
    const double* inv_in = nullptr;       // optional [T] 1/s_in, 1/s_full (IEEE quotients); else divided in-kernel
    const double* inv_full = nullptr;
    unsigned long long* peaks = nullptr;  // calibration recording [T][E] (FP mode)
};
// SpikeHook (quant.cpp:420-446): at seeded (sample, block, dir, t) positions,
// multiply `channels` hashed channels' b_bar by `gain`, before quantization.
struct SpikeCfg {
    double rate = 0.0;  // 0 = off
    double gain = 100.0;
    int channels = 1;   // <= kMaxSpikeChannels
    uint64_t salt = 0;
    int block = 0, dir = 0;
    int sample0 = 0;    // global index of this launch's sample 0
};
constexpr int kMaxSpikeChannels = 64;
struct ScanParams {
    int S = 0, T = 0, E = 0, N = 0;
    int order = 0, grid = 0;          // scan order of this direction
    const double* u = nullptr;        // [S][T][E] canonical scan input (conv output)
    const double* proj = nullptr;     // [S][T][E+2N] x_proj output rows in scan order (dpre | B | C)
    const double* a = nullptr;        // [E][N] continuous state matrix
    const double* b_delta = nullptr;  // [E]
    double* o = nullptr;              // [S][T][E] scan output at canonical positions
    int mode = MODE_DYNAMIC, n_refresh = 10, abits = 8, obits = 8;
    ScanKindCal cal[3];               // a_bar, b_bar, h
    const uint8_t* literal = nullptr; // [T] (device) 1 where the channel-local detector shortcut is not exact
    int literal_any = 0;              // host summary of `literal`
    int force_literal = 0;
    uint8_t* masks = nullptr;         // optional [3][S][T][E] O(t) after detection (parity)
    SpikeCfg spike;                   // reference-form kernel only (launch_scan)
};
cudaError_t launch_scan(const ScanParams& p, cudaStream_t st, bool* used_literal);
// Fast path (dynamic/static, channel-local detector): both directions in one
// launch (plus a step-table prep launch); work = scan_fast_workspace_bytes(S, T,
// ndirs) bytes, 16-aligned. variant 0: auto (the f32 state update on one thread
// per channel for A4 and even E, on two per channel otherwise); 1: the same with the
// certified f32 codes disabled (every element exact f64); 2: two threads per
// channel, f32 state; 3 / 4: one thread per channel with the f64 / f32 state update
// (even E); 5: two threads per channel, f64 state; 6: one thread per channel, f32
// state, in its large-grid shape (A in shared memory, 128 registers) at any size.
// Non-null `masks` selects the parity-trace instantiation.
// E > 0: also the small-batch split-phase scan's intermediates when S * E * ndirs
// is below one warp per SM (launch_scan_fast then uses that path in auto mode)
size_t scan_fast_workspace_bytes(int S, int T, int ndirs, int E = 0);
// merge (may be null): the out_proj input K1 (merge source), fused into the
// one-thread-per-channel f32-state kernel when that kernel runs (*merged = true;
// the caller has zeroed merge->ocnt; merge_cnt = [S][E/32] ints, zero between
// launches, left zero); otherwise the caller launches it.
cudaError_t launch_scan_fast(const ScanParams* dirs, int ndirs, void* work, size_t work_bytes, cudaStream_t st,
                             int variant, const K1Params* merge = nullptr, int* merge_cnt = nullptr,
                             bool* merged = nullptr);

// K4 auxiliaries.
cudaError_t launch_patch_gather(const double* img, double* patches, int S, int image, int channels, int patch,
                                cudaStream_t st);
cudaError_t launch_conv(const double* u0, const double* taps, double* u, int S, int T, int E, int W,
                        cudaStream_t st);
double measure_fp64_peak(cudaStream_t st, int num_sms);  // TFLOP/s (DFMA = 2 flops)
double measure_i8_peak(cudaStream_t st, int num_sms);    // dense int8 tensor TOP/s (tcgen05 kind::i8)
// fn: 0 exp, 1 log1p, 2 softplus, 3 silu (device forms, glibc-identical)
cudaError_t launch_math_eval(int fn, const double* x, double* y, size_t n, cudaStream_t st);
cudaError_t launch_meanpool(const double* x, double* pooled, int S, int T, int E, cudaStream_t st);

}  // namespace ob
