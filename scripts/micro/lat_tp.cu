// Latency / throughput probes for the instruction classes the K3 scan is made of
// (F2F f32<->f64, DMUL, DADD, DFMA, MUFU.EX2, LDS.64, I2F.F64), B200 sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_tp lat_tp.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N_IT 4096
template <int OP>
__global__ void lat(double* out, float* outf, int seed) {
    __shared__ double tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = threadIdx.x * 0.5;
    __syncthreads();
    double d = 1.0 + seed * 1e-9;
    float f = 1.0f + seed * 1e-7f;
    int k = seed & 7;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N_IT; ++i) {
        if (OP == 0) { f = __double2float_rn(d); d = static_cast<double>(f) * 1.0000001; }  // F2F pair + DMUL
        if (OP == 1) d = __dmul_rn(d, 1.0000001);
        if (OP == 2) d = __dadd_rn(d, 1e-9);
        if (OP == 3) d = __fma_rn(d, 1.0000001, 1e-9);
        if (OP == 4) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f)); f = y * 0.5f; }
        if (OP == 5) { d = tab[k]; k = static_cast<int>(d) & 31; }
        if (OP == 6) { f = static_cast<float>(d); d = static_cast<double>(f); }  // F2F.F32.F64 + F2F.F64.F32
        if (OP == 7) { f = f * 1.0000001f + 1e-9f; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) printf("op %d latency %.2f cycles/iter\n", OP, double(t1 - t0) / N_IT);
    out[threadIdx.x] = d + k;
    outf[threadIdx.x] = f;
}

// throughput: 8 independent chains per thread, many warps
template <int OP>
__global__ void tp(double* out, int seed) {
    double d[8];
    float f[8];
    int ki[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { d[j] = 1.0 + (seed + j) * 1e-9; f[j] = 1.0f + j * 1e-7f; ki[j] = j + seed; }
#pragma unroll 4
    for (int i = 0; i < 1024; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) f[j] = __double2float_rn(d[j] + f[j]);                  // DADD + F2F.F32.F64
            if (OP == 1) d[j] = static_cast<double>(f[j]), f[j] += 1.0f;          // F2F.F64.F32 + FADD
            if (OP == 2) d[j] = __dmul_rn(d[j], 1.0000001);
            if (OP == 3) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f[j])); f[j] = y; }
            if (OP == 4) d[j] = static_cast<double>(ki[j]), ki[j] += 3;           // I2F.F64 + IADD
            if (OP == 5) f[j] = f[j] * 1.0000001f;
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j] + f[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run_tp(double* out, int sms, const char* name, double elems_per_iter) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    tp<OP><<<sms * 8, 256>>>(out, 1);
    cudaEventRecord(a);
    tp<OP><<<sms * 8, 256>>>(out, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = double(sms) * 8 * 256 * 1024 * 8 * elems_per_iter;
    double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
    printf("%-28s %8.3f ms  %6.1f lane-ops/clk/SM (at %d MHz nominal)\n", name, ms, per_clk_sm, clk / 1000);
}

int main() {
    double* out; float* outf;
    cudaMalloc(&out, 1 << 26); cudaMalloc(&outf, 1 << 20);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    lat<0><<<1, 32>>>(out, outf, 1); lat<1><<<1, 32>>>(out, outf, 1); lat<2><<<1, 32>>>(out, outf, 1);
    lat<3><<<1, 32>>>(out, outf, 1); lat<4><<<1, 32>>>(out, outf, 1); lat<5><<<1, 32>>>(out, outf, 1);
    lat<6><<<1, 32>>>(out, outf, 1); lat<7><<<1, 32>>>(out, outf, 1);
    cudaDeviceSynchronize();
    run_tp<0>(out, sms, "DADD+F2F.F32.F64 (pairs)", 1);
    run_tp<1>(out, sms, "F2F.F64.F32+FADD (pairs)", 1);
    run_tp<2>(out, sms, "DMUL", 1);
    run_tp<3>(out, sms, "MUFU.EX2", 1);
    run_tp<4>(out, sms, "I2F.F64+IADD (pairs)", 1);
    run_tp<5>(out, sms, "FMUL", 1);
    cudaDeviceSynchronize();
    return 0;
}
