// Calibration: what a 32-byte-per-lane global store (STG.256) costs the L1TEX LSU data
// pipe when Q lanes of a warp cover one row's contiguous Q x 32 bytes (Q = 1: the
// lane-private pattern of k_zig_lst, 32 rows per instruction; Q = 4: a 128-byte line per
// quad, 8 rows per instruction; Q = 32: fully coalesced).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o calib_coop calib_coop.cu
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,gpu__time_duration.sum ./calib_coop
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

template <int Q>
__global__ void __launch_bounds__(768, 1) k_coop(int n_rows, int n_per, double* out)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int groups = n_rows / 32, gstride = gridDim.x * 24;
    uint64_t v = 0x9E3779B97F4A7C15ULL * (threadIdx.x + 1);
    // a group of 32 rows; per instruction the warp writes rows r0 .. r0 + 32/Q - 1, Q x 32 bytes each
    constexpr int RPI = 32 / Q;             // rows per instruction
    const int sub = lane / Q, part = lane % Q;
    for (int g = blockIdx.x * 24 + wib; g < groups; g += gstride) {
        double* base = out + (int64_t)g * 32 * n_per;
        for (int c = 0; c < n_per; c += 4 * Q) {      // columns covered by one pass over the group's rows
#pragma unroll
            for (int r0 = 0; r0 < 32; r0 += RPI) {
                double* dst = base + (int64_t)(r0 + sub) * n_per + c + 4 * part;
                v = v * 6364136223846793005ULL + 1;
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "l"(v), "l"(v ^ 1), "l"(v ^ 2), "l"(v ^ 3) : "memory");
            }
        }
    }
}

template <int Q>
void run(double* out, int n_rows, int n_per, int sms)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_coop<Q><<<sms, 768>>>(n_rows, n_per, out);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) k_coop<Q><<<sms, 768>>>(n_rows, n_per, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("Q=%2d: %.3f ms  %.0f GB/s  (%s)\n", Q, ms, (double)n_rows * n_per * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    const int n_rows = 1 << 22, n_per = 256;
    double* out; cudaMalloc(&out, (size_t)n_rows * n_per * 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1>(out, n_rows, n_per, sms);
    run<2>(out, n_rows, n_per, sms);
    run<4>(out, n_rows, n_per, sms);
    run<8>(out, n_rows, n_per, sms);
    run<32>(out, n_rows, n_per, sms);
    return 0;
}
