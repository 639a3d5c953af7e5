// Throughput of the polar pieces at full lane utilisation (calibration only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2405_19493_b200/csrc/gz_device.cuh"
#include "../../paper_2405_19493_b200/csrc/gz_libm.cuh"
__device__ uint64_t g_log_tab[256] = GZ_LOG_TAB_INIT;

// MODE 0: log only; 1: log+div+sqrt (polar multiplier); 2: LCG draws + v + s only; 3: cuda log()
template <int MODE>
__global__ void __launch_bounds__(256) k(int iters, double* out) {
    __shared__ uint64_t s_log[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_log[i] = g_log_tab[i];
    __syncthreads();
    uint64_t S = 0x123456789ULL + threadIdx.x * 77 + blockIdx.x * 7919;
    double acc = 0.0;
    double s = 0.25 + (threadIdx.x & 255) * 0.0025;   // main log branch (< 0.9375)
    for (int it = 0; it < iters; ++it) {
        if constexpr (MODE == 0) {
            acc += gz_log_t(s, s_log);
            s = __dadd_rn(s, 1e-9);
        } else if constexpr (MODE == 1) {
            const double mul = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, gz_log_t(s, s_log)), s));
            acc = __dadd_rn(acc, mul);
            s = __dadd_rn(s, 1e-9);
        } else if constexpr (MODE == 2) {
            const uint64_t t1 = 0x5DEECE66DULL * S + 0xB, t2 = 0x5DEECE66DULL * t1 + 0xB, t3 = 0x5DEECE66DULL * t2 + 0xB, t4 = 0x5DEECE66DULL * t3 + 0xB;
            S = t4;
            const uint64_t ua = ((uint64_t)(uint32_t)(t1 >> 16) << 32) | (uint32_t)(t2 >> 16);
            const uint64_t ub = ((uint64_t)(uint32_t)(t3 >> 16) << 32) | (uint32_t)(t4 >> 16);
            const double v1 = gz_unit53_pm1(ua), v2 = gz_unit53_pm1(ub);
            const double ss = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
            acc = (ss < 1.0) ? __dadd_rn(acc, ss) : acc;
        } else {
            acc += log(s);
            s = __dadd_rn(s, 1e-9);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, (size_t)sms * 16 * 256 * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    auto run = [&](auto kern, const char* name) {
        int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
        int grid = sms * occ;
        kern<<<grid, 256>>>(iters, out);
        cudaEventRecord(a);
        kern<<<grid, 256>>>(iters, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double n = (double)grid * 256 * iters;
        printf("%-22s occ=%d %.3f ms  %.1f G ops/s\n", name, occ, ms, n / ms / 1e6);
    };
    run(k<0>, "glibc-log (main)");
    run(k<1>, "polar multiplier");
    run(k<2>, "LCG attempt (4 steps)");
    run(k<3>, "cuda log()");
    return 0;
}
