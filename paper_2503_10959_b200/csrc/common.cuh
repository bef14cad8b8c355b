// Shared device helpers for the OuroMamba-Quant B200 kernels (sm_100a).
//
// All real-valued arithmetic on the hot path is IEEE f64 (B200 keeps a 1:2
// FP64:FP32 rate) with explicit __dmul_rn/__dadd_rn where the reference's
// operation order matters: the reference is built with -ffp-contract=off
// (/root/reference/proj/CMakeLists.txt:19-21), so products and sums are
// rounded separately and no FMA contraction may be introduced.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "glibc_math.cuh"

namespace ob {

constexpr int kMaxN = 16;  // state size N the scan keeps in registers

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// qmax_for(bits) = 2^(b-1) - 1, quant.cpp:15-18.
__host__ __device__ __forceinline__ double qmax_for(unsigned bits) {
    return static_cast<double>((1ll << (bits - 1)) - 1);
}

// quantize_code (quant.cpp:29-35) for a caller that already holds 1/s:
// clip(round_half_away(x / s), +-q) as a double, bit-identical to the
// reference. q2 = x * inv_s is within ~1.5 ulp of the exact quotient, so
// round-to-nearest of q2 equals round-half-away of the correctly rounded
// x / s unless q2 sits within a few ulp of a half-integer; only then is the
// IEEE division evaluated. |q2| is clamped first so the 1.5*2^52 rounding
// trick stays exact.
__device__ __forceinline__ double quant_code_inv(double x, double s, double inv_s, double q) {
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    double q2 = dmul(x, inv_s);
    q2 = fmin(fmax(q2, -(q + 1.0)), q + 1.0);
    double r = dadd(dadd(q2, kMagic), -kMagic);  // round to nearest (ties even)
    double d = dadd(q2, -r);
    if (fabs(d) > 0.4999999999990) {  // near a half-integer: decide exactly
        double qe = __ddiv_rn(x, s);
        r = round(qe);  // half away from zero, like std::round
    }
    return fmin(fmax(r, -q), q);
}

// quant_code_inv as an int, without the conversion pipe: 1.5*2^52 + r holds r
// in its low word (two's complement), the rest is quant_code_inv's test.
__device__ __forceinline__ int quant_code_int(double x, double s, double inv_s, double q, int qi) {
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    double q2 = dmul(x, inv_s);
    q2 = fmin(fmax(q2, -(q + 1.0)), q + 1.0);
    const double t = dadd(q2, kMagic);
    int c = __double2loint(t);
    if (fabs(dadd(q2, -dadd(t, -kMagic))) > 0.4999999999990) c = static_cast<int>(round(__ddiv_rn(x, s)));
    return min(max(c, -qi), qi);
}

// Same, exact division only (for per-channel outlier scales).
__device__ __forceinline__ double quant_code_div(double x, double s, double q) {
    double r = round(__ddiv_rn(x, s));
    return fmin(fmax(r, -q), q);
}

// scale_for(row, n, bits) = max|x| / q, or 1.0 for an all-zero row
// (quant.cpp:37-42), given the row peak.
__device__ __forceinline__ double scale_from_peak(double peak, double q) {
    return peak == 0.0 ? 1.0 : __ddiv_rn(peak, q);
}

// softplus_val / sigmoid_val / silu_val, tensor.hpp:146-154, with glibc's exp and
// log1p (glibc_math.cuh) so the values equal the reference's bit for bit.
__device__ __forceinline__ double softplus_d(double x) {
    return dadd(fmax(x, 0.0), gl::log1p(gl::exp(-fabs(x))));
}
__device__ __forceinline__ double sigmoid_d(double x) {
    if (x >= 0.0) return __ddiv_rn(1.0, dadd(1.0, gl::exp(-x)));
    double e = gl::exp(x);
    return __ddiv_rn(e, dadd(1.0, e));
}
__device__ __forceinline__ double silu_d(double x) { return dmul(x, sigmoid_d(x)); }

// maybe_refresh predicate (quant.cpp:303-311): clear before detection at t.
__host__ __device__ __forceinline__ bool refresh_at(int t, int n_refresh) {
    return n_refresh != 0 && t != 0 && (t % n_refresh) == 0;
}

// Scan permutation (ssm.cpp:30-46): canonical token visited at scan step t.
__host__ __device__ __forceinline__ int scan_perm(int order, int t, int grid) {
    int m = grid * grid, fast = t % grid, slow = t / grid;
    switch (order) {
        case 0: return slow * grid + fast;
        case 1: return m - 1 - (slow * grid + fast);
        case 2: return fast * grid + slow;
        default: return m - 1 - (fast * grid + slow);
    }
}

// Canonical row of scan step t for a sequence of T steps: identity (order <= 0),
// row-backward T-1-t (order 1), or the column orders of scan_perm (T = grid^2).
__host__ __device__ __forceinline__ int row_at(int order, int t, int T, int grid) {
    return order <= 0 ? t : (order == 1 ? T - 1 - t : scan_perm(order, t, grid));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace ob
