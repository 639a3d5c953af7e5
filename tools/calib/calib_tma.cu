// Calibration: the store side of the lane-per-stream kernels on B200.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o calib_tma calib_tma.cu
// Each warp owns 32 rows of an [n_rows][n_per] f64 array (C4 shape: 2^22 x 256)
// and produces one value per lane per iteration (an LCG48 draw converted to f64),
// staged in shared memory and written out by
//   mode 0: lanes (LDS + STG.128, 128-byte row segments, ring stride 33 doubles)
//   mode 1: one TMA tensor store per 16 columns (box 16 x 32, SWIZZLE_128B)
//   mode 2: two TMA tensor stores per 32 columns (256-byte row segments)
//   mode 3: four TMA tensor stores per 64 columns (512-byte row segments)
// and, separately, random 16-byte table gathers from shared memory with and
// without 8 replicas (one per 16-byte bank group).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t lcg2(uint64_t& S)
{
    const uint64_t t1 = (0x5DEECE66DULL * S + 0xBULL) & 0xffffffffffffULL;
    const uint64_t t2 = (0xBB20B4600A69ULL * S + 0x40942DE6BAULL) & 0xffffffffffffULL;
    S = t2;
    return ((t1 >> 16) << 32) | (t2 >> 16);
}

__device__ __forceinline__ void sts64(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory"); }

template <int MODE, int NW>
__global__ void __launch_bounds__(NW * 32) k_store(const __grid_constant__ CUtensorMap tm, int64_t n_rows, int n_per,
                                                   double* out, uint64_t seed)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    constexpr int TILE = 4096;                    // 32 rows x 16 doubles
    constexpr int NT = MODE == 3 ? 8 : 4;         // ring tiles per warp
    constexpr int FT = MODE == 1 ? 1 : MODE == 2 ? 2 : 4;   // tiles per flush
    unsigned char* ring = smem + (size_t)wib * (MODE == 0 ? 32 * 33 * 8 * 2 : NT * TILE);
    const uint32_t ring_sh = (uint32_t)__cvta_generic_to_shared(ring);
    const int64_t n_groups = n_rows / 32;
    for (int64_t grp = (int64_t)blockIdx.x * NW + wib; grp < n_groups; grp += (int64_t)gridDim.x * NW) {
        const int64_t row0 = grp * 32;
        uint64_t S = seed + row0 + lane;
        if constexpr (MODE == 0) {
            double* r = reinterpret_cast<double*>(ring);
            for (int f = 0; f < n_per; f += 16) {
                const int c0 = f & 31;
#pragma unroll 4
                for (int c = 0; c < 16; ++c) r[lane * 33 + c0 + c] = (double)(lcg2(S) >> 11);
                __syncwarp();
                const int q = lane & 7, rq = lane >> 3;
                double* base = out + (row0 + rq) * n_per + f + 2 * q;
#pragma unroll
                for (int it = 0; it < 8; ++it)
                    *reinterpret_cast<double2*>(base + (int64_t)it * 4 * n_per) =
                        make_double2(r[(rq + 4 * it) * 33 + c0 + 2 * q], r[(rq + 4 * it) * 33 + c0 + 2 * q + 1]);
                __syncwarp();
            }
        } else {
            int issued = 0;
            for (int f = 0; f < n_per; f += 16 * FT) {
                // wait until the tiles about to be written are no longer being read by TMA
                if (lane == 0 && issued >= NT / FT) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NT / FT - 1) : "memory");
                __syncwarp();
                for (int t = 0; t < FT; ++t) {
                    const int tile = ((f >> 4) + t) % NT;
                    const uint32_t tb = ring_sh + tile * TILE + lane * 128;
#pragma unroll 4
                    for (int c = 0; c < 16; ++c) {
                        const uint32_t off = ((((c >> 1) ^ (lane & 7)) << 4) | ((c & 1) << 3));
                        sts64(tb + off, (double)(lcg2(S) >> 11));
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    for (int t = 0; t < FT; ++t) {
                        const int tile = ((f >> 4) + t) % NT;
                        const int c0 = f + 16 * t, r0 = (int)row0;
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                                     ::"l"(&tm), "r"(c0), "r"(r0), "r"(ring_sh + tile * TILE) : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    ++issued;
                }
                issued = __shfl_sync(0xffffffffu, issued, 0);
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
        }
    }
    if (MODE != 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

/* mode 4: every lane copies its own row segment (SEG doubles) with a 1D bulk copy
   (cp.async.bulk, SASS UBLKCP) from a private padded ring row, no warp coupling */
template <int SEG, int NW>
__global__ void __launch_bounds__(NW * 32) k_lanebulk(int64_t n_rows, int n_per, double* out, uint64_t seed)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    constexpr int RS = 2 * SEG * 8 + 16;            /* ring row stride: two segments + 16 B pad */
    unsigned char* row = smem_raw + ((size_t)wib * 32 + lane) * RS;
    const uint32_t row_sh = (uint32_t)__cvta_generic_to_shared(row);
    const int64_t n_groups = n_rows / 32;
    for (int64_t grp = (int64_t)blockIdx.x * NW + wib; grp < n_groups; grp += (int64_t)gridDim.x * NW) {
        const int64_t r = grp * 32 + lane;
        uint64_t S = seed + r;
        int half = 0;
        for (int f = 0; f < n_per; f += SEG) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");   /* this half's previous copy */
            const uint32_t hb = row_sh + half * SEG * 8;
#pragma unroll 4
            for (int c = 0; c < SEG; ++c) sts64(hb + 8 * c, (double)(lcg2(S) >> 11));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + r * n_per + f),
                         "r"(hb), "n"(SEG * 8) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            half ^= 1;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int REP>
__global__ void __launch_bounds__(256) k_gather(const ulonglong2* tab, int iters, uint64_t* sink)
{
    __shared__ __align__(16) ulonglong2 s[128 * 8];
    for (int i = threadIdx.x; i < 128 * REP; i += blockDim.x) s[i] = tab[i / REP];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint64_t S = blockIdx.x * 256 + threadIdx.x + 1, acc = 0;
    for (int k = 0; k < iters; ++k) {
        const uint64_t u = lcg2(S);
        const uint32_t i = (uint32_t)(u >> 56) & 127u;
        const ulonglong2 v = s[REP == 1 ? i : i * REP + (lane & (REP - 1))];
        acc += v.x ^ v.y ^ u;
    }
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
}

int main()
{
    const int64_t n_rows = 1 << 22;
    const int n_per = 256;
    double* out;
    CK(cudaMalloc(&out, (size_t)n_rows * n_per * 8));
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)n_per, (cuuint64_t)n_rows};
    cuuint64_t strides[1] = {(cuuint64_t)n_per * 8};
    cuuint32_t box[2] = {16, 32}, es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](auto kern, int nw, size_t smem, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nw * 32, smem);
        const int grid = sms * occ;
        for (int w = 0; w < 3; ++w) kern<<<grid, nw * 32, smem>>>(tm, n_rows, n_per, out, 7);
        cudaEventRecord(e0);
        const int reps = 10;
        for (int w = 0; w < reps; ++w) kern<<<grid, nw * 32, smem>>>(tm, n_rows, n_per, out, 7 + w);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        printf("%-34s occ %d x %2d warps  %.3f ms  %.0f GB/s  %.1f G values/s  (%s)\n", name, occ, nw, ms,
               n_rows * n_per * 8.0 / ms / 1e6, n_rows * n_per / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    run(k_store<0, 8>, 8, 8 * 32 * 33 * 8 * 2 + 1024, "lanes STG.128 (128 B segments)");
    run(k_store<1, 8>, 8, 8 * 4 * 4096 + 1024, "TMA 16 cols/flush (128 B)");
    run(k_store<2, 8>, 8, 8 * 4 * 4096 + 1024, "TMA 32 cols/flush (256 B)");
    run(k_store<1, 4>, 4, 4 * 4 * 4096 + 1024, "TMA 16 cols/flush, 4-warp blocks");
    run(k_store<2, 4>, 4, 4 * 4 * 4096 + 1024, "TMA 32 cols/flush, 4-warp blocks");
    auto runl = [&](auto kern, int nw, size_t smem, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nw * 32, smem);
        const int grid = sms * occ;
        for (int w = 0; w < 3; ++w) kern<<<grid, nw * 32, smem>>>(n_rows, n_per, out, 7);
        cudaEventRecord(e0);
        for (int w = 0; w < 10; ++w) kern<<<grid, nw * 32, smem>>>(n_rows, n_per, out, 7 + w);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 10;
        printf("%-34s occ %d x %2d warps  %.3f ms  %.0f GB/s  %.1f G values/s  (%s)\n", name, occ, nw, ms,
               n_rows * n_per * 8.0 / ms / 1e6, n_rows * n_per / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    runl(k_lanebulk<16, 8>, 8, 8 * 32 * (2 * 16 * 8 + 16), "lane bulk 128 B, 8 warps");
    runl(k_lanebulk<32, 8>, 8, 8 * 32 * (2 * 32 * 8 + 16), "lane bulk 256 B, 8 warps");
    runl(k_lanebulk<32, 12>, 12, 12 * 32 * (2 * 32 * 8 + 16), "lane bulk 256 B, 12 warps");
    runl(k_lanebulk<32, 4>, 4, 4 * 32 * (2 * 32 * 8 + 16), "lane bulk 256 B, 4-warp blocks");
    runl(k_lanebulk<64, 4>, 4, 4 * 32 * (2 * 64 * 8 + 16), "lane bulk 512 B, 4-warp blocks");
    // table gathers
    std::vector<ulonglong2> h(128);
    for (int i = 0; i < 128; ++i) h[i] = make_ulonglong2(i * 0x9E3779B97F4A7C15ULL, i);
    ulonglong2* tab;
    uint64_t* sink;
    CK(cudaMalloc(&tab, 128 * 16));
    CK(cudaMalloc(&sink, (size_t)sms * 8 * 256 * 8));
    CK(cudaMemcpy(tab, h.data(), 128 * 16, cudaMemcpyHostToDevice));
    auto g = [&](auto kern, const char* name) {
        const int iters = 4096;
        kern<<<sms * 8, 256>>>(tab, iters, sink);
        cudaEventRecord(e0);
        kern<<<sms * 8, 256>>>(tab, iters, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-34s %.3f ms  %.1f G gathers/s\n", name, ms, (double)sms * 8 * 256 * iters / ms / 1e6);
    };
    g(k_gather<1>, "gather LDS.128, 1 copy");
    g(k_gather<8>, "gather LDS.128, 8 replicas");
    return 0;
}
