// f32 helpers of the fast scan's certified pre-pass (k3_scan_fast.cu), shared with
// tests/cpp/softplus_bound_check.cu, which checks the softplus bound exhaustively.
#pragma once

namespace ob {

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// f32 softplus(x) = max(x,0) + log1p(exp(-|x|)) and a bound eps on its relative
// error against the exact f64 softplus of the (double) argument that rounds to x:
// |softplus_f32(x) / softplus(x) - 1| <= eps = (kSoftplusEpsUnits + 3 max(0,-x)) 2^-24.
// e = ex2.approx(-|x| log2 e) (2^-22 plus the argument's rounding, 3|x| 2^-24
// relative); log1p(e) = 2 atanh(s), s = e / (2 + e) in (0, 1/3], by the odd series
// through s^13 (truncation < 0.3 x 2^-24 relative), __fdividef and six FMAs; one
// add; the double argument's rounding to f32 moves softplus by <= 2^-24 relative
// for x >= 0 and <= max(1, -x) 2^-24 for x < 0. tests/cpp/softplus_bound_check.cu evaluates every f32 x in [-80, 90]
// against the exact value and asserts the bound (largest ratio recorded there).
// Below x = -80 ex2.approx.ftz flushes; eps is then 1 (the exact path decides).
constexpr float kSoftplusEpsUnits = 12.0f;
__device__ __forceinline__ float softplus_f32(float x, float& eps) {
    const float e = ex2_approx(-fabsf(x) * 1.44269504f);
    eps = x < -80.0f ? 1.0f : fmaf(fmaxf(0.0f, -x), 3.0f, kSoftplusEpsUnits) * 5.9604645e-8f;
    const float sr = __fdividef(e, 2.0f + e), z = sr * sr;
    float pz = fmaf(z, 1.0f / 13.0f, 1.0f / 11.0f);
    pz = fmaf(z, pz, 1.0f / 9.0f);
    pz = fmaf(z, pz, 1.0f / 7.0f);
    pz = fmaf(z, pz, 1.0f / 5.0f);
    pz = fmaf(z, pz, 1.0f / 3.0f);
    pz = fmaf(z, pz, 1.0f);
    return fmaxf(x, 0.0f) + 2.0f * sr * pz;
}

}  // namespace ob
