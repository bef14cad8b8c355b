// Host engine of the B200 quantized VMM inference path: model weights and
// calibration tables resident in HBM, workspace sized per batch, and the
// forward as a fixed sequence of K1/K2/K3/K4 launches on one stream (captured
// into a CUDA graph per (batch, mode)).
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.h"

namespace ob {

// Error taxonomy of the reference (common.hpp:11-21 -> ouromamba.h:16-21).
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
inline void require(bool c, const std::string& m) {
    if (!c) throw ValidationError(m);
}
void cuda_check(cudaError_t e, const char* what);
// Process-wide counter bumped by every device (re)allocation or free of a
// DevBuf. A captured CUDA graph holds raw workspace/weight pointers, so the C
// ABI keys its graphs on this epoch and re-captures after any reallocation.
uint64_t alloc_epoch();
// Fresh id for a calibration's contents: assigned at creation and on every
// edit, so a graph never replays thresholds (passed by value) of an older version.
uint64_t next_calib_version();

struct Dims {  // ModelDims, ssm.hpp:42-56
    int image = 32, channels = 3, patch = 4, embed = 16, state = 4, blocks = 2, classes = 10, conv_width = 3;
    int grid() const { return image / patch; }
    int tokens() const { return grid() * grid(); }
    int patch_vals() const { return patch * patch * channels; }
};

struct QuantSpec {  // QuantSpec, quant.hpp:21-28
    unsigned wbits = 4, abits = 8, obits = 8;
    int n_refresh = 10;
    double rho = 0.01;
    void validate() const;
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release();
    void ensure(size_t count);  // grow-only
    void upload(const T* host, size_t count, cudaStream_t st);
};

struct QWeight {  // one W4 quant-linear operand
    int rows = 0, cols = 0;
    DevBuf<int8_t> codes, codes_t;  // [rows][cols], [cols][rows]
    DevBuf<double> scales;          // [rows]
};

class Context;

struct HostModel {  // ToyVmmModel tensors in f64 (ssm.hpp:58-66)
    Dims d;
    std::vector<int> orders;
    std::map<std::string, std::vector<double>> t;
    // W4 dequantized operand of a quantized weight (quantize_weights/dequantize_rows)
    std::vector<double> dequantized(const std::string& name, unsigned bits) const;
};
HostModel make_toy_model(const Dims& d, const std::vector<int>& orders, uint64_t seed);

struct TensorCal {
    double theta = 0.0;
    std::vector<double> s_in, s_full;
    std::vector<uint8_t> excluded;
};

class Calibration {
  public:
    QuantSpec spec;
    bool d1 = true, d2 = true;
    int tokens = 0, embed = 0, blocks = 0, ndirs = 0;
    std::vector<TensorCal> scan;  // [block][dir][kind]
    std::vector<TensorCal> lin;   // [block][site]
    int nsites() const { return ndirs + 2; }
    // device mirror
    DevBuf<double> dev;               // packed s_in/s_full tables
    DevBuf<uint8_t> literal;          // [block][dir][T]
    std::vector<int> literal_any;     // [block][dir]
    std::vector<int> lin_literal;     // [block][site]: some step fails the channel-local check
    bool dirty = true;
    uint64_t version = next_calib_version();
    void upload(cudaStream_t st);
    const double* s_in_dev(bool is_lin, size_t idx) const;
    const double* s_full_dev(bool is_lin, size_t idx) const;
    const double* inv_in_dev(bool is_lin, size_t idx) const;
    const double* inv_full_dev(bool is_lin, size_t idx) const;
};

// OURO tensor container (ouro_tensor.cpp; tensor_io.hpp:13-44).
enum class OuroDtype : uint32_t { F64 = 0, I8 = 1, U4 = 2 };
struct OuroTensor {
    std::vector<uint64_t> shape;
    OuroDtype dtype = OuroDtype::F64;
    std::string payload;  // bytes as stored (u4: nibble-packed)
};
void atomic_write_bytes(const std::string& path, const std::string& bytes);
std::string read_whole_file(const std::string& path);
size_t ouro_numel(const std::vector<uint64_t>& shape);
size_t ouro_payload_bytes(OuroDtype dt, const std::vector<uint64_t>& shape);
void pack_nibbles(const int8_t* codes, size_t n, uint8_t* out);     // (n + 1) / 2 bytes
void unpack_nibbles(const uint8_t* packed, size_t n, int8_t* out);  // n codes
void ouro_tensor_write(const std::string& path, OuroDtype dt, const std::vector<uint64_t>& shape, const void* payload,
                       size_t bytes);
OuroTensor ouro_tensor_read(const std::string& path);

// Calibration directories in the reference's format (calib_io.cpp).
void save_calibration_dir(const Calibration& c, int state, const std::string& dir);
void load_calibration_dir(Calibration& c, int state, const std::string& dir, bool want_d2);

class Model {
  public:
    Model(Context* ctx, HostModel hm);
    ~Model();
    Model(const Model&) = delete;
    Model& operator=(const Model&) = delete;
    Context* ctx;
    HostModel host;
    Dims d;
    // FP device weights
    DevBuf<double> patch_w, patch_b, head_w, head_b;
    struct DirDev {
        DevBuf<double> a, b_delta, xp;  // xp: (E+2N) x E = w_delta | w_b | w_c
    };
    struct BlockDev {
        DevBuf<double> w_inproj, conv, out_proj;  // w_inproj: 2E x E = w_in | w_gate
        std::vector<DirDev> dirs;
    };
    std::vector<BlockDev> blocks;
    // quantized weights (weight_bits); built on demand
    unsigned qbits = 0;
    DevBuf<double> patch_deq, head_deq;
    struct BlockQ {
        QWeight in, out;
        std::vector<QWeight> xp;
        DevBuf<double> conv_deq, in_deq, out_deq;
        std::vector<DevBuf<double>> xp_deq;
    };
    std::vector<BlockQ> qblocks;

    void set_tensor(const std::string& name, const double* data, size_t n);
    void upload_fp();
    void quantize(unsigned bits);
    bool fp_dirty = true;
    int k1_variant = 0;    // 0 auto (channel-parallel K1 wherever exact), 1 literal detector kernel,
                           // 2 auto with the register window kernel for plain / RMSNorm sources (A/B aid)
    int merge_fuse = 0;    // 1: the out_proj input K1 runs as the f32-state scan's tail (last direction of each
                           // (sample, channel group) to finish quantizes it); 0 (default): separate k1_channel
                           // launch. Measured at Vim-B batch 256: 3.36 ms scan per block fused vs 1.71 + 0.216
                           // separate (the tails walk 196 tokens per warp)
    int pack_a4 = 0;       // 1: A4 inlier codes travel nibble-packed from K1 to K2, which unpacks them in
                           // shared memory (QAct::codes4); 0 (default): one int8 byte per code. Measured at
                           // Vim-B batch 256: packed K2 176 / 107 / 127 us vs 157 / 93 / 119 (in_proj / x_proj /
                           // out_proj), forward +1.5 ms: the f64 outputs (260-560 MB per launch) bound K2, the
                           // packed operand saves 19 MB per launch and its unpack warpgroup adds ~4.5K
                           // warp-instructions per 128x128 tile
    SpikeCfg spikes;       // SpikeHook settings (rate 0 = off); block/dir set per scan
    int scan_variant = 0;  // 0 auto (fast path when exact), 1 per-direction reference kernel, 2 fast path, exact codes only,
                           // 3 fast path on the two-threads-per-channel kernel, 4 on the one-thread-per-channel kernel
                           // (f64 state update), 5 the one-thread-per-channel kernel with the f32 state update,
                           // 6 the two-threads-per-channel kernel with the f64 state update, 7 the
                           // one-thread f32-state kernel in its large-grid shape (A in shared memory)

    // workspace
    struct Work {
        int S = 0;
        DevBuf<double> x, patches, u0, gate, u, xin, pooled, logits, img;
        DevBuf<double> proj, o;  // per dir stacked
        DevBuf<int8_t> codes, ocode;
        DevBuf<double> s_row, oscale;
        DevBuf<int> ocnt;
        DevBuf<uint32_t> omask;
        DevBuf<uint8_t> scanned, masks, scan_steps, codes4;
        DevBuf<int> merge_cnt;  // [S][E/32] finish counters of the scan's fused merge K1 (zero between launches)
        DevBuf<unsigned long long> peaks;
        DevBuf<int32_t> acc_in, acc_out;
        std::vector<cudaEvent_t> feed_events;  // host-feed chunk events, created on first use
    } w;
    void ensure_work(Work& wk, int S, bool trace);
    // Split forward: a batch of >= parts * kSplitMin samples and >= parts * split_min_rows
    // token rows runs as `split_parts` independent sub-batches on their own streams
    // (samples never interact), so each part's kernels fill the others' last-wave tails.
    // Off for traces, calibration recording and per-family timing. Measured (ms per
    // forward, parts 1 / 2): Vim-B 224² batch 256 69.4 / 68.6, Vim-B 448² batch 64 73.9 /
    // 72.0 (50K rows each), Vim-S batch 64 12.12 / 12.76 (12.5K rows: smaller parts
    // lose more to their own tails than the overlap wins), hence 16K rows per part.
    static constexpr int kSplitMin = 32;
    static constexpr int kMaxSplit = 4;
    int split_parts = 2;
    int split_min_rows = 16384;
    int feed_chunks = 8;  // host-feed H2D chunks per forward (batches >= 64); e2e measured 2/4/8/16/32:
                          // 2599 / 2776 / 2795 / 2701 / 2682 images/s
    struct SplitPart {
        Work w;
        cudaStream_t st = nullptr, copy = nullptr;  // compute / H2D streams of parts >= 1
        cudaEvent_t fork = nullptr, join = nullptr;
    };
    SplitPart parts[kMaxSplit];

    // Per-kernel-family device time of one forward (CUDA events on the stream).
    enum Family { FAM_K1 = 0, FAM_K2 = 1, FAM_K3 = 2, FAM_DGEMM = 3, FAM_AUX = 4, FAM_COUNT = 5 };
    struct Timing {
        bool on = false;
        std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
        double ms[FAM_COUNT] = {0, 0, 0, 0, 0};
        int launches[FAM_COUNT] = {0, 0, 0, 0, 0};
        bool keep_list = false;
        long k0 = 0;  // kernel_launch_counter() at tick_begin
        std::vector<std::pair<int, double>> list;  // (family, ms) per launch, in order
    } timing;
    void tick_begin(int fam);
    void tick_end(int fam);
    void timing_collect();

    struct TraceSink {
        int block = -1;
        std::map<std::string, std::vector<char>> blobs;
    };
    // Runs the whole forward on `ctx` stream; images/logits are device pointers.
    // Host-image feed for the end-to-end call: the H2D copy of chunk k+1 (copy
    // stream) overlaps the patch gather + embedding of chunk k (main stream).
    struct HostFeed {
        const double* host = nullptr;  // pinned host images (B x pix)
        cudaStream_t copy = nullptr;
        int chunks = 1;
    };
    void forward(const Calibration* cal, int mode, bool d1, bool d2, const double* images, int S, double* logits,
                 TraceSink* trace, unsigned long long* calib_peaks, const HostFeed* feed = nullptr);
    // one (half-)batch on stream st with workspace wk (forward() validates and uploads first)
    void forward_impl(const Calibration* cal, int mode, bool d1, bool d2, const double* images, int S,
                      double* logits, TraceSink* trace, unsigned long long* calib_peaks, const HostFeed* feed,
                      cudaStream_t st, Work& w, int sample0 = 0);  // sample0: global index of sample 0 (SpikeHook)
    std::unique_ptr<Calibration> calibrate(const double* images_dev, int S, const QuantSpec& spec, bool d1, bool d2,
                                           int chunk);
};

class Context {
  public:
    explicit Context(int device);
    ~Context();
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    void set_stream(cudaStream_t s);
};

}  // namespace ob
