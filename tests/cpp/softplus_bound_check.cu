// Exhaustive check of the fast scan's f32 softplus bound (csrc/scan_f32.cuh):
// for every finite f32 x >= -80, (|softplus_f32(x) / softplus(x) - 1| + the
// argument-rounding term) / eps(x) must stay below 1, with
// softplus(x) the exact f64 value (glibc-identical exp/log1p). Prints the largest
// ratio and the x it occurs at; exit code 1 if the bound fails. The
// argument-rounding term is max(1, -x) 2^-24 for x < 0 and 2^-24 otherwise. GPU program, built
// and run by tests/test_gpu_f32_bounds.py.
#include <cstdio>
#include <cstdint>

#include "common.cuh"
#include "scan_f32.cuh"

__global__ void check(uint32_t lo, uint32_t hi, unsigned long long* worst) {
    double best = 0.0;
    uint32_t arg = 0;
    for (uint64_t b = lo + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b <= hi;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float x = __uint_as_float(static_cast<uint32_t>(b));
        float eps;
        const float a = ob::softplus_f32(x, eps);
        const double ex = ob::softplus_d(static_cast<double>(x));
        const double rel = fabs(static_cast<double>(a) / ex - 1.0);
        // the double argument's rounding to f32: sigma(x) |x| / softplus(x) <= 1 for x >= 0
        // (softplus(x) >= x) and <= |x| for x < 0 (softplus(x) >= sigma(x))
        const double var = (x < 0.0f ? fmax(1.0, -static_cast<double>(x)) : 1.0) * 0x1p-24 * 1.0001;
        const double r = (rel + var) / static_cast<double>(eps);
        if (r > best) {
            best = r;
            arg = static_cast<uint32_t>(b);
        }
    }
    // pack (ratio bits, argument) : ratios are positive, so their bits order like the values
    const unsigned long long key = (static_cast<unsigned long long>(__double_as_longlong(best)) & ~0xffffffffull) | arg;
    atomicMax(worst, key);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long));
    double worst = 0.0;
    float worst_x = 0.0f;
    // every finite x >= 0 and [-80, -0]: sign-magnitude ranges of f32 bit patterns
    const uint32_t ranges[2][2] = {{0x00000000u, 0x7F7FFFFFu}, {0x80000000u, 0xC2A00000u}};
    for (const auto& rg : ranges) {
        cudaMemset(d, 0, sizeof(unsigned long long));
        check<<<148 * 16, 256>>>(rg[0], rg[1], d);
        unsigned long long h = 0;
        cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
        const unsigned long long rb = h & ~0xffffffffull;
        double r;
        memcpy(&r, &rb, sizeof r);
        if (r >= worst) {
            worst = r;
            const uint32_t xb = static_cast<uint32_t>(h & 0xffffffffull);
            memcpy(&worst_x, &xb, sizeof worst_x);
        }
    }
    if (cudaGetLastError() != cudaSuccess) {
        printf("cuda error\n");
        return 2;
    }
    printf("worst_ratio %.6f at x = %.9g\n", worst, worst_x);
    return worst < 1.0 ? 0 : 1;
}
