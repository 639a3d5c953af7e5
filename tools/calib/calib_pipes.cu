// Pipe throughput micro-benchmarks (calibration only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(int iters, double* out, uint64_t* outi) {
    double a[8]; uint64_t b[8]; float f[8];
    for (int i = 0; i < 8; ++i) { a[i] = 1.0 + threadIdx.x * 1e-9 + i; b[i] = threadIdx.x + i; f[i] = 1.0f + i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (OP == 0) a[i] = __fma_rn(a[i], 0.999999, 1e-7);
            else if constexpr (OP == 1) b[i] = b[i] * 0x5DEECE66DULL + 0xB;      // 64-bit mad
            else if constexpr (OP == 2) f[i] = __fmaf_rn(f[i], 0.9999f, 1e-7f);
            else if constexpr (OP == 3) b[i] = (b[i] ^ (b[i] >> 7)) + 0x9E3779B9u; // 64-bit alu
            else a[i] = __dmul_rn(a[i], 0.999999);
        }
    }
    double s = 0; uint64_t si = 0;
    for (int i = 0; i < 8; ++i) { s += a[i] + f[i]; si ^= b[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s; outi[blockIdx.x * blockDim.x + threadIdx.x] = si;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out; uint64_t* outi; cudaMalloc(&out, sms * 8 * 256 * 8); cudaMalloc(&outi, sms * 8 * 256 * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 8192;
    auto run = [&](auto kern, const char* name) {
        int grid = sms * 8;
        kern<<<grid, 256>>>(iters, out, outi);
        cudaEventRecord(a);
        kern<<<grid, 256>>>(iters, out, outi);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)grid * 256 * iters * 8;
        printf("%-16s %.1f G lane-ops/s = %.1f per SM per clk (at %d MHz)\n", name, ops / ms / 1e6, ops / ms / 1e3 / sms / (clk / 1e3), clk / 1000);
    };
    run(k<0>, "DFMA");
    run(k<4>, "DMUL");
    run(k<2>, "FFMA");
    run(k<1>, "64-bit mad");
    run(k<3>, "64-bit alu mix");
    return 0;
}
