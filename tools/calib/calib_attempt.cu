// Ziggurat attempt-body throughput by stage (calibration only): which part of the
// lane attempt (LCG48 draw, layer split + table gather + compare, int->f64 and
// product, ring store) bounds the lane kernels.  Usage: calib_attempt
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void lcg2(uint32_t& lo, uint32_t& hi, uint32_t& uhi, uint32_t& ulo, uint64_t c1, uint64_t c2)
{
    const uint64_t p1 = (uint64_t)lo * 0xDEECE66Du + c1;
    const uint32_t t1h = (uint32_t)(p1 >> 32) + hi * 0xDEECE66Du + lo * 5u;
    const uint64_t p2 = (uint64_t)lo * 0xB4600A69u + c2;
    const uint32_t t2h = (uint32_t)(p2 >> 32) + hi * 0xB4600A69u + lo * 0xBB20u;
    uhi = __funnelshift_r((uint32_t)p1, t1h, 16);
    ulo = __funnelshift_r((uint32_t)p2, t2h, 16);
    lo = (uint32_t)p2;
    hi = t2h;
}

template <int STAGE, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(int rounds, const ulonglong2* tab, uint64_t* out, uint64_t c1, uint64_t c2)
{
    __shared__ __align__(16) ulonglong2 s_kw[128 * 8];
    extern __shared__ __align__(128) uint64_t ring[];
    for (int j = threadIdx.x; j < 1024; j += blockDim.x) s_kw[j] = tab[j / 8];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t lx = (uint32_t)(lane & 7) << 4;
    const char* kwb = reinterpret_cast<const char*>(s_kw) + lx;
    uint32_t lo = threadIdx.x * 7919u + blockIdx.x, hi = blockIdx.x;
    uint64_t acc = 0;
    uint32_t C = 0;
    for (int r = 0; r < rounds; ++r) {
        uint32_t fm = 0;
        uint64_t zbs[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            uint32_t uhi, ulo;
            lcg2(lo, hi, uhi, ulo, c1, c2);
            if constexpr (STAGE == 0) {
                acc ^= ((uint64_t)uhi << 32) | ulo;
                continue;
            }
            const uint32_t ioff = (uhi >> 17) & 0x3f80u;
            const ulonglong2 kw = *reinterpret_cast<const ulonglong2*>(kwb + ioff);
            const uint64_t m = ((uint64_t)(uhi & 0xffffffu) << 32) | ulo;
            if (m < kw.x) fm |= 1u << a;
            if constexpr (STAGE == 1) {
                acc += kw.y;
                continue;
            }
            const double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)kw.y));
            zbs[a] = (uint64_t)__double_as_longlong(x) ^ ((uint64_t)(uhi & 0x80000000u) << 32);
            if constexpr (STAGE == 2) acc ^= zbs[a];
        }
        if constexpr (STAGE >= 3) {
#pragma unroll
            for (int a = 0; a < 8; ++a) ring[threadIdx.x * 16 + ((C + a) & 15)] = zbs[a];
        }
        C += __ffs(~fm);
        acc += fm;
    }
    if constexpr (STAGE >= 3) acc ^= ring[threadIdx.x * 16 + (C & 15)];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + C;
}

int main()
{
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    ulonglong2 h[128];
    for (int i = 0; i < 128; ++i) h[i] = make_ulonglong2(i ? (0x00f0000000000000ull - i * 1000) : 0x00e0000000000000ull, 0x3c90000000000000ull + i);
    ulonglong2* tab; uint64_t* out;
    cudaMalloc(&tab, sizeof h); cudaMemcpy(tab, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMalloc(&out, (size_t)sms * 1024 * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int rounds = 4096;
    auto run = [&](auto kern, int nw, const char* name) {
        const int dyn = nw * 32 * 16 * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        kern<<<sms, nw * 32, dyn>>>(rounds, tab, out, 0xB, 0x40942DE6BAull);
        cudaEventRecord(a);
        kern<<<sms, nw * 32, dyn>>>(rounds, tab, out, 0xB, 0x40942DE6BAull);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double att = (double)sms * nw * 32 * rounds * 8;
        printf("%-28s warps/SM %2d: %7.1f G attempts/s  %.2f per SM per clk\n", name, nw, att / ms / 1e6, att / ms / 1e3 / sms / (clk / 1e3));
    };
#define RUNS(ST, NAME) run(k<ST, 8>, 8, NAME); run(k<ST, 16>, 16, NAME); run(k<ST, 24>, 24, NAME); run(k<ST, 32>, 32, NAME);
    RUNS(0, "LCG48 draw")
    RUNS(1, "+ split, gather, compare")
    RUNS(2, "+ int->f64, product, sign")
    RUNS(3, "+ ring stores")
    return 0;
}
