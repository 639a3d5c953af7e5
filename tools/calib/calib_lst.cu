// Calibration: the store pattern of k_zig_lst on B200 (no generation work).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o calib_lst calib_lst.cu
// [n_rows][n_per] f64 output (C4 shape: 2^22 x 256), lane l of warp g owns rows
// (g + k * warps) * 32 + l, one after the other, and writes each row front to back
// with per-lane stores of CH bytes (16: STG.128, 32: STG.256, 64 / 128: 2 / 4 x STG.256
// back to back).  SKEW > 0 staggers the lanes' columns (lane l starts its first row
// l * SKEW deviates late), as the drift of the generating kernel does.
// k_lane_rmw: the config-5 mutation pattern -- each lane reads its row in 32-byte chunks
// (ld.global.v4.b64, PF chunks ahead in registers) and writes every chunk back updated.
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

template <int PF, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_lane_rmw(int n_rows, int n_per, double* out, int gens)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int groups = n_rows / 32, gstride = gridDim.x * NW;
    const int g0 = blockIdx.x * NW + wib;
    const int ng = g0 < groups ? (groups - g0 + gstride - 1) / gstride : 0;
    const int64_t per_row = (int64_t)n_per * gens;       /* a row is visited gens times */
    const int64_t total = (int64_t)ng * per_row;
    uint64_t b[PF][4];
    auto addr = [&](int64_t w) {
        const int k = (int)(w / per_row), c = (int)(w % per_row) % n_per;
        return out + ((int64_t)(g0 + k * gstride) * 32 + lane) * n_per + c;
    };
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        const int64_t w = 4 * j;
        if (w < total) asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(b[j][0]), "=l"(b[j][1]), "=l"(b[j][2]), "=l"(b[j][3]) : "l"(addr(w)));
    }
    for (int64_t w = 0; w < total; w += 4 * PF) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const int64_t wj = w + 4 * j;
            if (wj < total) {
                double* d = addr(wj);
                const uint64_t v0 = b[j][0] + 1, v1 = b[j][1] + 1, v2 = b[j][2] + 1, v3 = b[j][3] + 1;
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(d), "l"(v0), "l"(v1), "l"(v2), "l"(v3) : "memory");
                const int64_t wn = wj + 4 * PF;
                if (wn < total) asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(b[j][0]), "=l"(b[j][1]), "=l"(b[j][2]), "=l"(b[j][3]) : "l"(addr(wn)) : "memory");
            }
        }
    }
}

template <int PF, int NW>
int run_rmw(double* out, int n_rows, int n_per, int sms, int gens)
{
    auto k = k_lane_rmw<PF, NW>;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) k<<<sms, NW * 32>>>(n_rows, n_per, out, gens);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    const int reps = 5;
    for (int i = 0; i < reps; ++i) k<<<sms, NW * 32>>>(n_rows, n_per, out, gens);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double bytes = (double)n_rows * n_per * gens * 16;
    printf("rmw PF %d  warps/SM %2d  rows %d x %d x %d gens: %.3f ms  %.0f GB/s  (%.1f G updates/s)\n", PF, NW, n_rows, n_per,
           gens, ms, bytes / ms / 1e6, bytes / 16 / ms / 1e6);
    return 0;
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
    run_rmw<2, 24>(out, 65536, 1024, sms, 10);
    run_rmw<4, 24>(out, 65536, 1024, sms, 10);
    run_rmw<4, 16>(out, 65536, 1024, sms, 10);
    run_rmw<8, 16>(out, 65536, 1024, sms, 10);
    run_rmw<4, 32>(out, 65536, 1024, sms, 10);
    for (int skew : {0, 4}) {
        run<16, 24>(out, n_rows, n_per, sms, skew);
        run<32, 24>(out, n_rows, n_per, sms, skew);
        run<32, 16>(out, n_rows, n_per, sms, skew);
        run<32, 32>(out, n_rows, n_per, sms, skew);
        if (skew == 0) run<64, 24>(out, n_rows, n_per, sms, skew);
        if (skew == 0) run<128, 24>(out, n_rows, n_per, sms, skew);
    }
    return 0;
}
