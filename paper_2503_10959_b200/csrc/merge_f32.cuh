// The merge source's certified f32 form (k1_detect_quant.cu), shared with
// tests/cpp/merge_bound_check.cu, which checks its bound exhaustively in g.
#pragma once

namespace ob {

// Merge source, certified form. v = m * silu(g) with m = (0 + o_0) + o_1 exact
// in f64; v is evaluated in f32 with a relative error bound, and the detector
// decision and inlier code are taken from it only when the bound keeps them
// away from theta and from half-integers; otherwise (and for outlier channels)
// the exact f64 value is used. Bound (derivation; tests/cpp/merge_bound_check.cu
// evaluates every f32 g >= -80 and asserts it): g and m rounded to f32 (2 x 2^-24),
// the ex2 argument (3|g| 2^-24 relative in e), ex2.approx (2^-22), the
// sigmoid's add (2^-24) and its quotient by __fdividef (2 ulp <= 4 x 2^-24 for
// a denominator in [1, 2]), both doubled for g < 0 where e/(1+e) carries e's
// error in full, two products: |vf/v - 1| <= (6|g| + 21) 2^-24, inside the
// (6|g| + 24) 2^-24 the kernel uses; the code adds 1/s rounded to f32 and one
// product. Below g = -80 ex2 flushes, so those elements always take the exact
// path.
struct MergeApprox {
    float v, eps;
};
__device__ __forceinline__ MergeApprox merge_approx(double m, double g) {
    const float gf = __double2float_rn(g), mf = __double2float_rn(m);
    const float ag = fabsf(gf);
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-ag * 1.44269504f));
    const float den = 1.0f + e;
    const float sig = __fdividef(gf >= 0.0f ? 1.0f : e, den);
    MergeApprox r;
    r.v = (mf * gf) * sig;
    if (m == 0.0 || g == 0.0) {  // v = +-0 exactly: code 0, never an outlier (frequent: all-zero h codes)
        r.v = 0.0f;
        r.eps = 0.0f;
        return r;
    }
    // f32 subnormals (relative error unbounded), the ex2 flush and overflow take the exact path
    const bool ok = gf >= -80.0f && ag >= 1e-30f && fabsf(mf) >= 1e-30f && fabsf(r.v) < 1e30f;
    r.eps = ok ? fmaf(ag, 6.0f, 24.0f) * 5.9604645e-8f : 1.0f;
    return r;
}

}  // namespace ob
