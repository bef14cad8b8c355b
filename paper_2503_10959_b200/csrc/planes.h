// K1 over streams of K x C planes and the GPU-backed gemm-bench stage
// (planes.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "kernels.h"

namespace ob {

// detect_outliers + split_quantize over steps planes x[t][ch][i] (K channels x
// C values), outlier state carried across steps with maybe_refresh(n_refresh).
// Output: the QAct operand of K2 with rows r = t*C + i and Kp >= K channels
// (codes 0 beyond K). work: plane_workspace_bytes(steps, K) bytes.
struct PlaneParams {
    const double* x = nullptr;
    int steps = 0, K = 0, Kp = 0, C = 0;
    double theta = 0.0;
    const double* s_in = nullptr;  // [steps] S^I(t)
    int n_refresh = 0, abits = 4, obits = 8;
    QAct a;
    uint8_t* scanned = nullptr;  // optional [steps] DetectResult::scanned
    int* count_out = nullptr;    // optional [steps] |O(t)| after detection
    void* work = nullptr;
};
size_t plane_workspace_bytes(int steps, int K);
cudaError_t launch_detect_planes(const PlaneParams& p, cudaStream_t st);

// gemm.hpp:103-138
struct SweepSettings {
    std::vector<size_t> periods = {1, 5, 10, 20, 0};  // 0 = never refresh
    size_t steps = 300;
    size_t m = 8, k = 512, c = 32;
    size_t persistent_channels = 6;
    double transient_rate = 0.15;
    double spike_gain = 40.0;
    size_t trials = 5;
    uint64_t seed = 1;
};
struct SweepRecord {
    size_t period = 0;
    double median_total_ns = 0.0;
    double mean_o_list = 0.0;
    double scans_per_step = 0.0;
};
struct BenchSettings {
    std::vector<size_t> sizes = {64, 128, 256};
    double outlier_fraction = 0.01;
    size_t trials = 5;
    uint64_t seed = 1;
    bool f16_output = false;
};
struct BenchRecord {
    std::string path;  // "hybrid" or "f64"
    size_t size = 0;
    double median_ns = 0.0;
};
// outputs (optional): every period's GEMM outputs, [period][step][column][m]
std::vector<SweepRecord> refresh_sweep(const SweepSettings& s, cudaStream_t st, int num_sms,
                                       std::vector<double>* outputs);
std::vector<BenchRecord> gemm_bench(const BenchSettings& s, cudaStream_t st, int num_sms);

}  // namespace ob
