// Calibration: the store pattern of k_zig_lst on B200 (no generation work).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o calib_lst calib_lst.cu
// [n_rows][n_per] f64 output (C4 shape: 2^22 x 256), lane l of warp g owns rows
// (g + k * warps) * 32 + l, one after the other, and writes each row front to back
// with per-lane stores of CH bytes (16: STG.128, 32: STG.256, 64 / 128: 2 / 4 x STG.256
// back to back).  SKEW > 0 staggers the lanes' columns (lane l starts its first row
// l * SKEW deviates late), as the drift of the generating kernel does.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int CH, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_lane_rows(int n_rows, int n_per, double* out, int skew)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int groups = n_rows / 32, gstride = gridDim.x * NW;
    const int g0 = blockIdx.x * NW + wib;
    const int ng = g0 < groups ? (groups - g0 + gstride - 1) / gstride : 0;
    const int64_t total = (int64_t)ng * n_per;          /* deviates of the lane over all its rows */
    constexpr int D = CH / 8;                            /* deviates per store burst */
    uint64_t v = 0x9E3779B97F4A7C15ULL * (threadIdx.x + 1);
    for (int64_t w = -(int64_t)lane * skew; w < total + 31 * skew; w += D) {
        if (w < 0 || w >= total) continue;
        const int k = (int)(w / n_per), c = (int)(w % n_per);
        double* dst = out + ((int64_t)(g0 + k * gstride) * 32 + lane) * n_per + c;
        v = v * 6364136223846793005ULL + 1;
        if constexpr (D == 2) {
            asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(dst), "l"(v), "l"(v ^ 1) : "memory");
        } else {
#pragma unroll
            for (int j = 0; j < D / 4; ++j)
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * j), "l"(v), "l"(v ^ 1), "l"(v ^ 2),
                             "l"(v ^ j)
                             : "memory");
        }
    }
}

template <int CH, int NW>
int run(double* out, int n_rows, int n_per, int sms, int skew)
{
    auto k = k_lane_rows<CH, NW>;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k<<<sms, NW * 32>>>(n_rows, n_per, out, skew);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) k<<<sms, NW * 32>>>(n_rows, n_per, out, skew);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double bytes = (double)n_rows * n_per * 8;
    printf("CH %3d B  warps/SM %2d  skew %3d: %.3f ms  %.0f GB/s  (%.1f G deviates/s)\n", CH, NW, skew, ms,
           bytes / ms / 1e6, bytes / 8 / ms / 1e6);
    return 0;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n_rows = 1 << 22, n_per = 256;
    double* out;
    CK(cudaMalloc(&out, (size_t)n_rows * n_per * 8));
    for (int skew : {0, 4, 37}) {
        run<16, 24>(out, n_rows, n_per, sms, skew);
        run<32, 24>(out, n_rows, n_per, sms, skew);
        run<32, 16>(out, n_rows, n_per, sms, skew);
        run<32, 32>(out, n_rows, n_per, sms, skew);
        run<64, 24>(out, n_rows, n_per, sms, skew);
        run<128, 24>(out, n_rows, n_per, sms, skew);
    }
    return 0;
}
