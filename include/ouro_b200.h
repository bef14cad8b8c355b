#ifndef OURO_B200_H
#define OURO_B200_H

/*
 * C ABI of the B200-native OuroMamba-Quant inference path (sm_100a).
 *
 * Drop-in boundary for the reference's hot path. Conventions follow the
 * reference C interface (/root/reference/proj/include/ouromamba.h):
 *   - every call returns an ouro_status; on failure ouro_b200_last_error()
 *     holds a thread-local message, cleared by the next successful call
 *     (ouromamba.h:28-29, src/capi.cpp:14-37);
 *   - NULL handles / pointers are rejected with OURO_ERR_VALIDATION, never a
 *     crash; _free(NULL) is a no-op (tests/test_capi.cpp:85-114);
 *   - handles are opaque; no global state besides the per-thread error
 *     message, so independent contexts may be used from different threads
 *     (ouromamba.h:4-10).
 * CUDA launch-configuration errors map to OURO_ERR_VALIDATION, device faults
 * to OURO_ERR_NUMERIC. Device pointers ("dev") must live on the context's
 * device; all operator calls are asynchronous on the context's stream.
 * INTEGRATION.md shows the binding a reference maintainer would add.
 */

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef OURO_STATUS_DEFINED
#define OURO_STATUS_DEFINED
typedef enum ouro_status {
    OURO_OK = 0,
    OURO_ERR_VALIDATION = 2, /* bad arguments, config or shapes */
    OURO_ERR_NUMERIC = 3,    /* device fault / non-finite values */
    OURO_ERR_IO = 4          /* missing, unreadable or unwritable files */
} ouro_status;
#endif

typedef struct ouro_b200_ctx ouro_b200_ctx;
typedef struct ouro_b200_model ouro_b200_model;
typedef struct ouro_b200_calib ouro_b200_calib;
typedef struct ouro_b200_trace ouro_b200_trace;

/* Quantization modes (quant.hpp:101): FP = bypass (no activation quantization). */
enum { OURO_B200_MODE_FP = 0, OURO_B200_MODE_DYNAMIC = 1, OURO_B200_MODE_STATIC = 2 };
/* Quant-linear epilogue post-ops. */
enum { OURO_B200_POST_STORE = 0, OURO_B200_POST_INPROJ = 1, OURO_B200_POST_RESID = 2, OURO_B200_POST_BIAS = 3,
       OURO_B200_POST_XPROJ = 4 /* first `split` columns: softplus(y + bias[r]) */ };
/* K1 row sources. */
enum { OURO_B200_SRC_PLAIN = 0, OURO_B200_SRC_RMSNORM = 1, OURO_B200_SRC_MERGE = 2 };

const char* ouro_b200_version(void);
const char* ouro_b200_last_error(void);

/* ---- context --------------------------------------------------------------- */
ouro_status ouro_b200_ctx_create(int device, ouro_b200_ctx** out);
void ouro_b200_ctx_free(ouro_b200_ctx* ctx);
/* Run on a caller stream (cudaStream_t, e.g. torch.cuda.current_stream()). */
ouro_status ouro_b200_ctx_set_stream(ouro_b200_ctx* ctx, void* stream);
ouro_status ouro_b200_ctx_synchronize(ouro_b200_ctx* ctx);
ouro_status ouro_b200_ctx_num_sms(ouro_b200_ctx* ctx, int* out);

/* ---- operator level (device pointers) ---------------------------------------- */

/* K1: per-step dynamic outlier detector + activation quantizer over S
 * sequences of T (sample, token) planes of E channels. Replaces, per plane,
 * maybe_refresh + detect_outliers (quant.hpp:67-80, quant.cpp:303-335) and
 * split_quantize (gemm.hpp:51-57, gemm.cpp:106-135).
 *   x      dev f64 [S][T][E] canonical rows (SRC_MERGE: scan output of dir 0)
 *   x2     dev f64 [S][T][E] scan output of dir 1 (SRC_MERGE, may be NULL)
 *   gate   dev f64 [S][T][E] (SRC_MERGE)
 *   order  scan order read at step t (ssm.cpp:30-46), -1 = identity; grid = sqrt(T)
 *   s_in, s_full  dev f64 [T] calibrated per-step scales (TensorCalib, quant.hpp:36-42)
 *   literal  1 = run the verbatim detector (cross-channel max per plane); 0 =
 *          channel-parallel kernel, exact when fl(nextafter(theta)/q_a) > s_in[t]
 *          for every t (the caller checks), unless `scanned`
 *          is requested; 2 = the channel-parallel path on the register window
 *          kernel for SRC_PLAIN / SRC_RMSNORM where E % 64 == 0 and E <= 768
 *          (A/B aid; 0 runs the bulk-copy staged kernel)
 * Outputs (row = s*T + t, dev): codes int8 [S*T][E] (0 at outliers), s_row
 * f64 [S*T], ocnt int32 [S*T] = |O(t)|, omask uint32 [S*T][ceil(E/32)]
 * (bit ch%32 of word ch/32 = channel in O(t)), ocode int8 / oscale f64
 * [S*T][E] written at outlier positions only, optional scanned uint8 [S*T]
 * (DetectResult::scanned; literal kernel). rs_work: ignored (kept for ABI
 * stability; the staged kernel computes D1 row factors in shared memory), may
 * be NULL. */
ouro_status ouro_b200_detect_quantize(ouro_b200_ctx* ctx, const double* x, const double* x2, const double* gate,
                                      size_t S, size_t T, size_t E, int src, int order, int grid, double theta,
                                      const double* s_in, const double* s_full, size_t n_refresh, unsigned act_bits,
                                      unsigned outlier_bits, int mode, int literal, int8_t* codes, double* s_row,
                                      int32_t* ocnt, uint32_t* omask, int8_t* ocode, double* oscale,
                                      uint8_t* scanned, double* rs_work);

/* K1 with the A4 inlier codes nibble-packed (pack_int4's layout, gemm.cpp:60-73 / PackedInt4,
 * gemm.hpp:40-49, with the channels as its columns: byte [m][ch/2], low nibble = even channel),
 * act_bits = 4, E even: codes4 dev uint8 [S*T][E/2]. Every other argument as
 * ouro_b200_detect_quantize. */
ouro_status ouro_b200_detect_quantize_packed(ouro_b200_ctx* ctx, const double* x, const double* x2, const double* gate,
                                             size_t S, size_t T, size_t E, int src, int order, int grid, double theta,
                                             const double* s_in, const double* s_full, size_t n_refresh,
                                             unsigned outlier_bits, int mode, int literal, uint8_t* codes4,
                                             double* s_row, int32_t* ocnt, uint32_t* omask, int8_t* ocode,
                                             double* oscale, uint8_t* scanned);

/* K2: hybrid quant-linear on tcgen05 kind::i8 (hybrid_gemm, gemm.hpp:78-87,
 * gemm.cpp:181-225): out[m][r] = ws[r]*(s_row[m]*acc_in[m][r]
 *   + sum_{ch in O(m), ascending} (oscale[m][ch]*w[r][ch])*ocode[m][ch]),
 * then the post-op. The activation operand is K1's output (M rows of K
 * channels); w dev int8 [R][K] weight codes (|code| <= 7), wt its transpose
 * [K][R]; ws dev f64 [R] weight row scales. K must be a multiple of 16 and R
 * of 32; acc_in and acc_out are requested together.
 * acc_in/acc_out (dev int32 [M][R], may be NULL) receive the reference's
 * integer planes GemmResult::acc_inlier / acc_outlier. */
ouro_status ouro_b200_quant_linear(ouro_b200_ctx* ctx, size_t M, size_t R, size_t K, const int8_t* codes,
                                   const double* s_row, const int32_t* ocnt, const uint32_t* omask,
                                   const int8_t* ocode, const double* oscale, const int8_t* w, const int8_t* wt,
                                   const double* ws, int post, double* out, size_t ld_out, double* out2, size_t split,
                                   const double* bias, int32_t* acc_in, int32_t* acc_out);

/* K2 on the nibble-packed A4 operand of ouro_b200_detect_quantize_packed (codes4 dev uint8
 * [M][K/2], K a multiple of 32): the packed tiles are loaded by TMA and expanded to int8
 * in shared memory before the tcgen05 MMA (gemm_i4 unpacks per call, gemm.cpp:142-143).
 * Every other argument and every output as ouro_b200_quant_linear. */
ouro_status ouro_b200_quant_linear_packed(ouro_b200_ctx* ctx, size_t M, size_t R, size_t K, const uint8_t* codes4,
                                          const double* s_row, const int32_t* ocnt, const uint32_t* omask,
                                          const int8_t* ocode, const double* oscale, const int8_t* w,
                                          const int8_t* wt, const double* ws, int post, double* out, size_t ld_out,
                                          double* out2, size_t split, const double* bias, int32_t* acc_in,
                                          int32_t* acc_out);

/* K3: selective scan of one direction with the QuantHook policy (s6_scan,
 * ssm.hpp:131-132, ssm.cpp:124-186; QuantHook quant.cpp:456-501), N = 16.
 *   u     dev f64 [S][T][E] canonical scan input; proj dev f64 [S][T][E+2N]
 *         rows in scan order = (delta pre-activation | B | C), the x_proj
 *         quant-linear output; delta = softplus(dpre + b_delta) in-kernel
 *   a     dev f64 [E][N]; b_delta dev f64 [E]; o dev f64 [S][T][E] (canonical)
 *   theta[3], s_in[3], s_full[3]: calibration of a_bar, b_bar, h (s_* dev [T])
 *   literal dev uint8 [T] (may be NULL): steps where the channel-local detector
 *   is not exact; force_literal runs the literal detector on every step.
 *   masks dev uint8 [3][S][T][E] (may be NULL): O(t) per kind after detection. */
ouro_status ouro_b200_quant_scan(ouro_b200_ctx* ctx, size_t S, size_t T, size_t E, size_t N, int order, int grid,
                                 const double* u, const double* proj, const double* a, const double* b_delta,
                                 double* o, int mode, size_t n_refresh, unsigned act_bits, unsigned outlier_bits,
                                 const double* theta, const double* const* s_in, const double* const* s_full,
                                 const uint8_t* literal, int force_literal, uint8_t* masks);

/* f64 projection with the reference's per-output k-ascending order
 * (detail::mm, tensor.cpp:373-382): out[m][r] = 0.0 + sum_k a[m][k]*w[r][k]. */
ouro_status ouro_b200_dgemm(ouro_b200_ctx* ctx, size_t M, size_t R, size_t K, const double* a, size_t lda,
                            const double* w, int post, double* out, size_t ld_out, double* out2, size_t split,
                            const double* bias);

/* ---- model level ---------------------------------------------------------------- */

/* dims = {image, channels, patch, embed, state, blocks, classes, conv_width}
 * (ModelDims, ssm.hpp:42-56); orders = ScanOrder values (ssm.hpp:15).
 * Weights are seeded exactly as make_toy_model (ssm.cpp:88-120). */
ouro_status ouro_b200_model_create(ouro_b200_ctx* ctx, const size_t* dims, const int* orders, size_t ndirs,
                                   uint64_t seed, ouro_b200_model** out);
void ouro_b200_model_free(ouro_b200_model* m);
/* Names as the reference checkpoint (ssm.cpp:381-405): "patch_embed.w"-style
 * names use this repo's spelling: patch_w, patch_b, head_w, head_b,
 * block<b>.{w_in,w_gate,conv,out_proj}, block<b>.dir<d>.{a,w_b,w_c,w_delta,b_delta}. */
ouro_status ouro_b200_model_set_tensor(ouro_b200_model* m, const char* name, const double* host, size_t n);
ouro_status ouro_b200_model_get_tensor(ouro_b200_model* m, const char* name, double* host, size_t cap,
                                       size_t* n_out);

/* Calibration (CalibrationResult, quant.hpp:44-49) extended with the
 * linear-input sites of D2. which: 0 = scan tensors [block][dir][kind],
 * 1 = linear sites [block][site]. Arrays are host memory. */
ouro_status ouro_b200_calib_create(ouro_b200_model* m, const unsigned* bits /* w,a,o */, size_t n_refresh,
                                   double rho, int d1, int d2, ouro_b200_calib** out);
ouro_status ouro_b200_calibrate(ouro_b200_model* m, const double* images_dev, size_t B, const unsigned* bits,
                                size_t n_refresh, double rho, int d1, int d2, size_t chunk, ouro_b200_calib** out);
void ouro_b200_calib_free(ouro_b200_calib* c);
/* Dequantized weight operand (quantize_weights + dequantize_rows,
 * quant.cpp:355-384) at `bits`: "patch_w", "head_w", "block<b>.in" (w_in|w_gate),
 * "block<b>.out_proj", "block<b>.conv", "block<b>.dir<d>.xp" (w_delta|w_b|w_c).
 * out == NULL queries the size into *n. Host memory. */
ouro_status ouro_b200_model_get_qweight(ouro_b200_model* m, const char* name, unsigned bits, double* out,
                                       size_t cap, size_t* n);

/* Calibration directories in the reference's on-disk format
 * (save_calibration / load_calibration, quant.cpp:179-290): calibration.txt
 * plus one <name>_scales.ouro f64 [2][tokens] file per scan tensor
 * block<b>.dir<d>.{a_bar,b_bar,h}. The D2 linear-site tables go to
 * d2_linear_sites.txt (+ scale files), which the reference ignores. Load
 * checks the directory against the model's dims; d2 = 1 needs the D2 file
 * (a reference-written directory loads with d2 = 0). Missing or malformed
 * files -> OURO_ERR_IO. */
ouro_status ouro_b200_calib_save(ouro_b200_calib* c, ouro_b200_model* m, const char* dir);
ouro_status ouro_b200_calib_load(ouro_b200_model* m, const char* dir, int d1, int d2, ouro_b200_calib** out);
/* The spec a calibration carries: bits = {weight, act, outlier}, n_refresh, rho, d1, d2. */
ouro_status ouro_b200_calib_spec(ouro_b200_calib* c, unsigned* bits, size_t* n_refresh, double* rho, int* d1,
                                 int* d2);

ouro_status ouro_b200_calib_count(ouro_b200_calib* c, int which, size_t* out);
ouro_status ouro_b200_calib_get(ouro_b200_calib* c, int which, size_t idx, double* theta, double* s_in,
                                double* s_full, uint8_t* excluded);
ouro_status ouro_b200_calib_set(ouro_b200_calib* c, int which, size_t idx, double theta, const double* s_in,
                                const double* s_full, const uint8_t* excluded);

/* Quantized (or FP) Vim forward: images dev f64 [B][image][image][channels],
 * logits dev f64 [B][classes]. d1 = pre-norm residual, d2 = quantized linear
 * inputs. Asynchronous on the context stream. */
ouro_status ouro_b200_forward(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                              const double* images_dev, size_t B, double* logits_dev);
/* Same through host buffers: H2D of the images and D2H of the logits inside
 * the call (synchronous). */
ouro_status ouro_b200_forward_host(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                   const double* images_host, size_t B, double* logits_host);
/* Capture CUDA graphs of ouro_b200_forward for repeated calls with the same
 * (calib, mode, d1, d2, images, B, logits) (1 = on). */
ouro_status ouro_b200_model_use_graphs(ouro_b200_model* m, int on);

/* Engine options: "scan_variant" = 0 auto (fast K3 path wherever the
 * channel-local detector is exact), 1 per-direction reference scan kernel,
 * 2 fast path with every a_bar/b_bar code computed in exact f64 (test aid),
 * 3 / 4 / 5 / 6 fast path on two threads per channel (f32 state) / one thread
 * per channel (f64 state) / one thread per channel (f32 state) / two threads per
 * channel (f64 state) (A/B aid); 7 the one-thread f32-state kernel in its
 * large-grid shape (A in shared memory) at any size (test aid);
 * "k1_variant" = 0 auto (channel-parallel K1 wherever exact), 1 literal
 * detector kernel everywhere, 2 auto with the register window plain / RMSNorm
 * kernel (A/B aid); "pack_a4" = 1: A4 activation codes travel
 * nibble-packed from K1 to K2, 0 (default) one int8 byte per code; "merge_fuse" = 1:
 * the out_proj input K1 runs as the f32-state scan's tail, 0 (default) its own
 * launch; "split_parts" in [1, 4] (default 2) runs a batch of
 * >= 32 * parts samples and >= parts * "split_min_rows" (default 16384) token
 * rows as that many independent sub-batches on their own streams (results
 * identical), 1 one stream; "feed_chunks" (default 8) = H2D chunks of
 * forward_host for batches >= 64. */
ouro_status ouro_b200_model_set_option(ouro_b200_model* m, const char* key, long value);

/* One forward with CUDA events around every launch: per kernel family
 * {K1 detect/quantize, K2 quant-linear, K3 scan, f64 projection, aux} the
 * summed device milliseconds (ms[5]) and launch counts (launches[5]). */
ouro_status ouro_b200_forward_profile(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                      const double* images_dev, size_t B, double* logits_dev, double* ms,
                                      int* launches);

/* Same, one entry per launch in issue order: family[k] (0-4 as above) and
 * ms[k]; *n = number of launches (entries beyond cap are dropped). */
ouro_status ouro_b200_forward_profile_launches(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                               const double* images_dev, size_t B, double* logits_dev, double* ms,
                                               int* family, size_t cap, size_t* n);

/* Measured FP64 FMA throughput of this device (TFLOP/s, 2 flops per DFMA),
 * the roofline denominator of the f64 scan (no vendor figure is used). */
ouro_status ouro_b200_measure_fp64_peak(ouro_b200_ctx* ctx, double* tflops);

/* Measured dense int8 tensor throughput (TOP/s, 2 ops per MAC) of this device:
 * back-to-back tcgen05.mma.kind::i8 M=128 N=256 K=32 on every SM, the K2
 * roofline denominator. */
ouro_status ouro_b200_measure_i8_peak(ouro_b200_ctx* ctx, double* tops);

/* Number of this library's kernels launched so far by the calling host thread
 * (every launcher counts its <<<>>> launches; CUDA-graph replays are not
 * host launches and do not count). The delta over one eager forward is the
 * kernels per step a graph replay of that forward launches (bench.py
 * `gpu_launches`). */
ouro_status ouro_b200_launch_count(long long* out);

/* Spike injection (SpikeSettings / SpikeHook, quant.hpp:105-118,
 * quant.cpp:420-446): at (sample, block, dir, t) positions chosen by the
 * reference's mix64 chain with probability `rate`, `channels` hashed channels'
 * b_bar values are multiplied by `gain` before quantization. rate 0 = off;
 * channels in [1, 64]. */
typedef struct {
    double rate, gain;
    size_t channels;
    uint64_t salt;
    size_t sample0; /* global index of the call's first sample (a batch sharded across GPUs) */
} ouro_b200_spikes;
/* Spikes for every later forward / trace of this model (NULL = off); spiked
 * scans run on the reference-form kernel. Cached graphs are rebuilt. */
ouro_status ouro_b200_model_set_spikes(ouro_b200_model* m, const ouro_b200_spikes* spikes);
/* quant_scan with spikes: block, dir and the global index of sample 0 place the
 * scan in the reference's StepContext (quant.cpp:559). */
ouro_status ouro_b200_quant_scan_spiked(ouro_b200_ctx* ctx, size_t S, size_t T, size_t E, size_t N, int order,
                                        int grid, const double* u, const double* proj, const double* a,
                                        const double* b_delta, double* o, int mode, size_t n_refresh,
                                        unsigned act_bits, unsigned outlier_bits, const double* theta,
                                        const double* const* s_in, const double* const* s_full,
                                        const ouro_b200_spikes* spikes, size_t block, size_t dir, size_t sample0);

/* detect_outliers + split_quantize over a stream of `steps` planes of K
 * channels x C values, x dev f64 [steps][K][C] (channel = row of the plane,
 * quant.cpp:313-335, gemm.cpp:106-135): maybe_refresh(t, n_refresh) clears the
 * outlier list, a channel's peak is its max |x| over the C values, the scan
 * fires when max_{ch not in O} peak / q(act_bits) > s_in[t] and then adds every
 * channel with peak > theta; inlier values are coded at s_in[t], outlier
 * channels at their own scale peak / q(outlier_bits). Outputs are the K2
 * operand with rows r = t*C + i and channel stride Kp >= K (codes 0 beyond K):
 * codes int8 [steps*C][Kp], s_row f64, ocnt int32 (|O(t)|), omask uint32
 * [steps*C][ceil(Kp/32)], ocode int8 / oscale f64 [steps*C][Kp] at outlier
 * positions, optional scanned uint8 [steps] (DetectResult::scanned). K <= 4096. */
ouro_status ouro_b200_detect_quantize_planes(ouro_b200_ctx* ctx, const double* x, size_t steps, size_t K, size_t C,
                                             double theta, const double* s_in, size_t n_refresh, unsigned act_bits,
                                             unsigned outlier_bits, size_t Kp, int8_t* codes, double* s_row,
                                             int32_t* ocnt, uint32_t* omask, int8_t* ocode, double* oscale,
                                             uint8_t* scanned);

/* The gemm-bench stage on the GPU (run_gemm_bench, pipeline.cpp:229-275).
 * Settings and records mirror SweepSettings / SweepRecord / BenchSettings /
 * BenchRecord (gemm.hpp:103-138); operands are drawn exactly as the
 * reference's bench_refresh_sweep / bench_gemm draw them from `seed`, so
 * mean_o_list and scans_per_step equal the reference's. Times are device time
 * (CUDA events) per trial, median over trials: the sweep times the plane
 * detector + quantizer and one K2 launch over all steps per period; the bench
 * times K2 ("hybrid", path 0) and the f64 GEMM of the dequantized operands
 * ("f64", path 1). `outputs` (nullable): the sweep's GEMM outputs,
 * [n_periods][steps][c][m] (the reference's y[m][c] per step). */
typedef struct {
    const size_t* periods; /* 0 = never refresh */
    size_t n_periods;
    size_t steps, m, k, c, persistent_channels;
    double transient_rate, spike_gain;
    size_t trials;
    uint64_t seed;
} ouro_b200_sweep_settings;
typedef struct {
    size_t period;
    double median_total_ns, mean_o_list, scans_per_step;
} ouro_b200_sweep_record;
ouro_status ouro_b200_refresh_sweep(ouro_b200_ctx* ctx, const ouro_b200_sweep_settings* s,
                                    ouro_b200_sweep_record* records, double* outputs);
typedef struct {
    const size_t* sizes;
    size_t n_sizes;
    double outlier_fraction;
    size_t trials;
    uint64_t seed;
    int f16_output;
} ouro_b200_bench_settings;
typedef struct {
    int path; /* 0 hybrid, 1 f64 */
    size_t size;
    double median_ns;
} ouro_b200_bench_record;
/* records: 2 * n_sizes entries, per size hybrid then f64 */
ouro_status ouro_b200_gemm_bench(ouro_b200_ctx* ctx, const ouro_b200_bench_settings* s,
                                 ouro_b200_bench_record* records);

/* ---- OURO tensor files (tensor_io.hpp:13-44) -----------
 * The reference's container: "OURO" | u32 version 1 | u32 rank | u64 dims |
 * u32 dtype | payload, little-endian. dtype: */
enum { OURO_B200_DTYPE_F64 = 0, OURO_B200_DTYPE_I8 = 1, OURO_B200_DTYPE_U4 = 2 };
/* write_tensor_f64 / _i8 / _u4 (tensor_io.cpp): data = f64[numel], int8[numel],
 * or for U4 either int8 codes in [-8, 7] (data_packed = 0: packed here, element
 * i in the low nibble of byte i/2 when i is even) or the packed payload itself
 * (data_packed = 1, ceil(numel/2) bytes, e.g. the codes4 operand of
 * ouro_b200_detect_quantize_packed copied from the device). Written atomically
 * (temporary file + rename). A code outside [-8, 7] is a validation error. */
ouro_status ouro_b200_tensor_save(const char* path, int dtype, const uint64_t* shape, size_t rank, const void* data,
                                  int data_packed);
/* Header of a tensor file: dtype, rank and the first `cap` dims (shape may be
 * NULL). Missing file, bad magic / version / dtype tag, truncation -> IO. */
ouro_status ouro_b200_tensor_info(const char* path, int* dtype, uint64_t* shape, size_t cap, size_t* rank);
/* Payload of a tensor file whose dtype must equal `dtype` (else IO, "dtype
 * mismatch", as read_tensor_*): f64 / int8 elements, or for U4 the codes
 * sign-extended to int8 (out_packed = 0, read_tensor_u4) or the packed bytes
 * (out_packed = 1). cap = capacity of `out` in bytes. */
ouro_status ouro_b200_tensor_load(const char* path, int dtype, void* out, size_t cap, int out_packed);

/* ---- Pipeline stages on the GPU (ouromamba.h:58-65, capi.cpp:166-186) ------
 * The settings a stage reads from the reference's RunConfig (config.hpp:17-47;
 * the text parser itself is out of scope). Scan orders are
 * row-forward, row-backward. run_id tags the metrics lines (the reference uses
 * the FNV-1a hash of its canonical config text, run_id_of; NULL = "b200").
 * d1 = d2 = 0 is the reference's own quantized pass. */
typedef struct {
    size_t image, channels, patch, embed, state, blocks, classes, conv_width; /* [model] */
    uint64_t seed;
    unsigned weight_bits, act_bits, outlier_bits; /* [quant] */
    size_t n_refresh;                             /* 0 = never ("full") */
    double outlier_quantile;                      /* rho */
    const char* mode;                             /* "dynamic", "static" or "bypass" */
    size_t eval_batch;
    double spike_rate, spike_gain;
    size_t spike_channels;
    int d1, d2; /* declared extensions */
    const char* run_id;
    int device;
} ouro_b200_stage_config;
/* run_quant_eval (pipeline.cpp:115-167): make_toy_model(dims, seed), the
 * calibration directory (its quantization settings must equal the config's),
 * the first min(B, eval_batch) images of `images_file` (OURO f64 [B, H*W*C]);
 * quantized_forward's metrics on the GPU (logits_mse, argmax_agreement, the
 * teacher-forced mse_block<b>.dir<d>, and in dynamic mode the QuantHook timeline
 * of sample 0's b_bar tensors) written to out_dir/metrics.txt in the
 * reference's line format ("run=<id> stage=quant-eval k=v ...", "%.17g"), plus
 * out_dir/manifest.txt. */
ouro_status ouro_b200_quant_eval(const ouro_b200_stage_config* cfg, const char* calib_dir, const char* images_file,
                                 const char* out_dir);
/* run_calib (pipeline.cpp:100-113): GPU calibration of the images in
 * `images_file` written as the reference's calibration directory (plus the D2
 * tables when cfg->d2) and a manifest. */
ouro_status ouro_b200_calib_stage(const ouro_b200_stage_config* cfg, const char* images_file, const char* out_dir);

/* Diagnostic: y[i] = f(x[i]) on the device for the path's transcendental
 * functions, fn = 0 exp, 1 log1p, 2 softplus, 3 silu (tensor.hpp:146-154);
 * x and y are device pointers of n doubles. The device forms restate glibc's
 * exp/log1p so they equal the reference's std::exp/std::log1p bit for bit;
 * the tests hold them to that against the host libm. */
ouro_status ouro_b200_math_eval(ouro_b200_ctx* ctx, int fn, const double* x_dev, double* y_dev, size_t n);

/* Parity harness: run a forward over host images and keep every
 * intermediate of one block (keys documented in DESIGN.md §5). */
ouro_status ouro_b200_trace_run(ouro_b200_model* m, ouro_b200_calib* c, int mode, int d1, int d2,
                                const double* images_host, size_t B, size_t block, ouro_b200_trace** out);
ouro_status ouro_b200_trace_get(ouro_b200_trace* t, const char* key, void* host, size_t cap, size_t* bytes);
void ouro_b200_trace_free(ouro_b200_trace* t);

#ifdef __cplusplus
}
#endif

#endif /* OURO_B200_H */
