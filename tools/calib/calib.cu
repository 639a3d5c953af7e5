// Calibration micro-kernels: where does the lane-per-stream ziggurat spend its time?
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o calib calib.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2405_19493_b200/csrc/gz_device.cuh"

constexpr int WARPS = 8;

template <int LK, int LSTRIDE, int LRING>
__device__ __forceinline__ void flushK(const double* ring, double* out, int64_t ld, int64_t row0, int f, int c0, int lane) {
    constexpr int LPR = LK / 2;            // lanes per row (16 B each)
    constexpr int RPI = 32 / LPR;          // rows per instruction
    const int q = lane % LPR, rq = lane / LPR;
    double* base = out + (row0 + rq) * ld + f + 2 * q;
    int ca = c0 + 2 * q; if (ca >= LRING) ca -= LRING;
    int cb = ca + 1; if (cb >= LRING) cb -= LRING;
    const double* src = ring + rq * LSTRIDE;
#pragma unroll
    for (int it = 0; it < 32 / RPI; ++it)
        *reinterpret_cast<double2*>(base + (int64_t)(it * RPI) * ld) = make_double2(src[it * RPI * LSTRIDE + ca], src[it * RPI * LSTRIDE + cb]);
}

// MODE 0: staging only (value = w); 1: + LCG draw -> double; 2: + table lookup/compare (always accept);
// 3: direct (uncoalesced) stores instead of staging, with LCG draw
template <int MODE, int LK, int LRING, int NW, int OCC>
__global__ void __launch_bounds__(NW * 32, OCC) k(int64_t n_streams, int n_per, const uint64_t* st_in, double* out, const ulonglong2* kwg) {
    extern __shared__ __align__(16) unsigned char smem[];
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(smem);
    double* s_ring = reinterpret_cast<double*>(smem + 16 * 128);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_kw[i] = kwg[i];
    __syncthreads();
    constexpr int LSTRIDE = LRING + 1;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* ring = s_ring + wib * 32 * LSTRIDE;
    double* myring = ring + lane * LSTRIDE;
    const int64_t n_groups = (n_streams + 31) >> 5;
    for (int64_t grp = (int64_t)blockIdx.x * NW + wib; grp < n_groups; grp += (int64_t)gridDim.x * NW) {
        const int64_t row0 = grp * 32, sid = row0 + lane;
        uint64_t S = st_in[sid];
        int w = 0, flushed = 0, wslot = 0, fslot = 0;
        while (flushed < n_per) {
            const int lim = min(n_per, flushed + LRING);
#pragma unroll 2
            for (int it = 0; it < LK; ++it) {   // (wrap of the ring row handled by the flush reading contiguous LK)
                if (w < lim) {
                    double v;
                    if constexpr (MODE == 0) {
                        v = (double)w;
                    } else {
                        const uint64_t t1 = gz_lcg_mad(GZ_LCG_A, S, GZ_LCG_C);
                        const uint64_t t2 = gz_lcg_mad(0xBB20B4600A69ULL, S, 0x40942DE6BAULL);
                        S = t2;
                        const uint64_t u = gz_lcg_u64(t1, t2);
                        if constexpr (MODE == 1 || MODE == 3) {
                            v = __ull2double_rn(u & 0xffffffffffffffULL);
                        } else {
                            const uint32_t i = (uint32_t)(u >> 56) & 127u;
                            const uint64_t m = u & 0xffffffffffffffULL;
                            const ulonglong2 kw = s_kw[i];
                            const double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)kw.y));
                            v = (m < kw.x) ? x : -x;
                        }
                    }
                    if constexpr (MODE == 3) out[sid * (int64_t)n_per + w] = v;
                    else myring[wslot] = v;
                    ++w;
                    wslot = (wslot + 1 == LRING) ? 0 : wslot + 1;
                }
            }
            if constexpr (MODE != 3) {
                __syncwarp();
                flushK<LK, LSTRIDE, LRING>(ring, out, n_per, row0, flushed, fslot, lane);
                fslot = (fslot + LK >= LRING) ? fslot + LK - LRING : fslot + LK;
                __syncwarp();
            }
            flushed += LK;
        }
        st_in += 0;
    }
}

// pure coalesced store bandwidth: each warp writes its rows contiguously
__global__ void k_store(int64_t n, double* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<double2*>(out)[i] = make_double2((double)i, 1.0);
}

int main() {
    const int64_t n_streams = 1 << 22; const int n_per = 256;
    uint64_t* st; double* out; ulonglong2* kw;
    cudaMalloc(&st, n_streams * 8); cudaMemset(st, 1, n_streams * 8);
    cudaMalloc(&out, n_streams * n_per * 8);
    cudaMalloc(&kw, 128 * 16); cudaMemset(kw, 0x7f, 128 * 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto run = [&](auto kern, const char* name, int lring, int nw) {
        const size_t smem = 16 * 128 + nw * 32 * (lring + 1) * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nw * 32, smem);
        int grid = sms * occ;
        for (int r = 0; r < 2; ++r) kern<<<grid, nw * 32, smem>>>(n_streams, n_per, st, out, kw);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) kern<<<grid, nw * 32, smem>>>(n_streams, n_per, st, out, kw);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("%-28s occ=%d  %.3f ms  %.1f Gvar/s  %.0f GB/s  err=%s\n", name, occ, ms, n_streams * n_per / ms / 1e6,
               n_streams * n_per * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    run(k<0, 16, 32, 8, 1>, "stage LK16 R32 8w", 32, 8);
    run(k<2, 16, 32, 8, 1>, "lcg  LK16 R32 8w", 32, 8);
    run(k<0, 32, 40, 6, 1>, "stage LK32 R40 6w", 40, 6);
    run(k<2, 32, 40, 6, 1>, "lcg  LK32 R40 6w", 40, 6);
    run(k<0, 32, 48, 4, 1>, "stage LK32 R48 4w", 48, 4);
    run(k<2, 32, 48, 4, 1>, "lcg  LK32 R48 4w", 48, 4);
    run(k<0, 32, 64, 4, 1>, "stage LK32 R64 4w", 64, 4);
    run(k<2, 32, 64, 4, 1>, "lcg  LK32 R64 4w", 64, 4);
    run(k<0, 64, 72, 2, 1>, "stage LK64 R72 2w", 72, 2);
    run(k<2, 64, 72, 2, 1>, "lcg  LK64 R72 2w", 72, 2);
    {
        int grid = sms * 8;
        k_store<<<grid, 256>>>(n_streams * n_per, out);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_store<<<grid, 256>>>(n_streams * n_per, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("%-28s %.3f ms  %.0f GB/s\n", "store-only 16B coalesced", ms, n_streams * n_per * 8 / ms / 1e6);
    }
    return 0;
}
