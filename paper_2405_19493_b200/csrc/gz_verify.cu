/*
 * gz_verify.cu -- on-device verification statistics over generated deviates
 * (SURVEY 8f row 1 and row 3): the step right after generation in the
 * reference's `verify`/`bits` commands (cli.py:147-208, 239-256), which there
 * run as Python loops over host arrays.
 *
 *   gz_hist_edges    counts per bin for sorted interior edges with
 *                    numpy.searchsorted(edges, x, side="right") semantics
 *                    (stats.py:276-315 chi_square_gof binning)
 *   gz_ks_stat       two-sided Kolmogorov-Smirnov D against the standard normal
 *                    CDF 0.5*erfc(-x/sqrt 2) (stats.py:262-273): device radix sort
 *                    (CUB) + per-element D+/D- + max reduction
 *   gz_lowbits_hist  histogram of the low k bits of u64 draws
 *                    (stats.py:334-353 low_bits_chi_square)
 * Integer counts are exact; D uses CUDA's erfc (within a few ulp of glibc's).
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_radix_sort.cuh>

#include "../../include/gz_b200.h"

namespace {

constexpr int HIST_MAX_BINS = 4096;

__global__ void __launch_bounds__(256) k_hist_edges(const double* __restrict__ x, int64_t n,
                                                    const double* __restrict__ edges, int n_edges,
                                                    unsigned long long* counts)
{
    extern __shared__ unsigned char smem[];
    double* s_e = reinterpret_cast<double*>(smem);
    unsigned int* s_c = reinterpret_cast<unsigned int*>(smem + 8 * n_edges);
    for (int i = threadIdx.x; i < n_edges; i += blockDim.x) s_e[i] = edges[i];
    for (int i = threadIdx.x; i <= n_edges; i += blockDim.x) s_c[i] = 0;
    __syncthreads();
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[k];
        int lo = 0, hi = n_edges;          /* number of edges <= v */
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_e[mid] <= v) lo = mid + 1; else hi = mid;
        }
        atomicAdd(&s_c[lo], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= n_edges; i += blockDim.x)
        if (s_c[i]) atomicAdd(&counts[i], (unsigned long long)s_c[i]);
}

__global__ void __launch_bounds__(256) k_lowbits(const uint64_t* __restrict__ x, int64_t n, int k_bits,
                                                 unsigned long long* counts)
{
    __shared__ unsigned int s_c[256];
    const uint32_t cells = 1u << k_bits;
    for (uint32_t i = threadIdx.x; i < cells; i += blockDim.x) s_c[i] = 0;
    __syncthreads();
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&s_c[(uint32_t)x[k] & (cells - 1u)], 1u);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cells; i += blockDim.x)
        if (s_c[i]) atomicAdd(&counts[i], (unsigned long long)s_c[i]);
}

/* ordered-bits encoding of a non-negative double for atomicMax on u64 */
__device__ __forceinline__ unsigned long long ord(double d)
{
    return (unsigned long long)__double_as_longlong(d);
}

/* D+ = max(i/n - F(x_(i))), D- = max(F(x_(i)) - (i-1)/n) over the sorted sample */
__global__ void __launch_bounds__(256) k_ks(const double* __restrict__ xs, int64_t n, unsigned long long* dpm)
{
    double dp = 0.0, dm = 0.0;
    const double nn = (double)n;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double F = 0.5 * erfc(-xs[k] * 0.7071067811865475244);
        const double i = (double)(k + 1);
        dp = fmax(dp, i / nn - F);
        dm = fmax(dm, F - (i - 1.0) / nn);
    }
    for (int o = 16; o > 0; o >>= 1) {
        dp = fmax(dp, __shfl_xor_sync(0xffffffffu, dp, o));
        dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&dpm[0], ord(dp));   /* D+ and D- are >= 0 */
        atomicMax(&dpm[1], ord(dm));
    }
}

int sms_of_current()
{
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

} // namespace

extern "C" {

int gz_hist_edges(const double* x, int64_t n, const double* edges, int n_edges, uint64_t* counts, void* cuda_stream)
{
    if (n < 0 || n_edges < 1 || n_edges >= HIST_MAX_BINS || !counts || !edges) return GZ_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (cudaMemsetAsync(counts, 0, (size_t)(n_edges + 1) * 8, s) != cudaSuccess) return GZ_ERR_CUDA;
    if (n == 0) return GZ_OK;
    const size_t smem = 8 * (size_t)n_edges + 4 * (size_t)(n_edges + 1);
    const int grid = (int)((n + 255) / 256 < (int64_t)sms_of_current() * 8 ? (n + 255) / 256 : sms_of_current() * 8);
    k_hist_edges<<<grid, 256, smem, s>>>(x, n, edges, n_edges, (unsigned long long*)counts);
    return cudaGetLastError() == cudaSuccess ? GZ_OK : GZ_ERR_CUDA;
}

int gz_lowbits_hist(const uint64_t* x, int64_t n, int k_bits, uint64_t* counts, void* cuda_stream)
{
    if (n < 0 || k_bits < 1 || k_bits > 8 || !counts) return GZ_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (cudaMemsetAsync(counts, 0, (size_t)(1 << k_bits) * 8, s) != cudaSuccess) return GZ_ERR_CUDA;
    if (n == 0) return GZ_OK;
    const int grid = (int)((n + 255) / 256 < (int64_t)sms_of_current() * 8 ? (n + 255) / 256 : sms_of_current() * 8);
    k_lowbits<<<grid, 256, 0, s>>>(x, n, k_bits, (unsigned long long*)counts);
    return cudaGetLastError() == cudaSuccess ? GZ_OK : GZ_ERR_CUDA;
}

int gz_ks_stat(const double* x, int64_t n, double* d_out, void* cuda_stream)
{
    if (n < 1 || n > (1ll << 31) - 1 || !x || !d_out) return GZ_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    double* sorted = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    unsigned long long* dpm = nullptr;
    int st = GZ_OK;
    if (cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, x, (double*)nullptr, (int)n, 0, 64, s) != cudaSuccess)
        return GZ_ERR_CUDA;
    if (cudaMallocAsync((void**)&sorted, (size_t)n * 8, s) != cudaSuccess ||
        cudaMallocAsync(&tmp, tmp_bytes, s) != cudaSuccess || cudaMallocAsync((void**)&dpm, 16, s) != cudaSuccess) {
        st = GZ_ERR_CUDA;
    } else if (cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, x, sorted, (int)n, 0, 64, s) != cudaSuccess ||
               cudaMemsetAsync(dpm, 0, 16, s) != cudaSuccess) {
        st = GZ_ERR_CUDA;
    } else {
        const int grid = (int)((n + 255) / 256 < (int64_t)sms_of_current() * 8 ? (n + 255) / 256 : sms_of_current() * 8);
        k_ks<<<grid, 256, 0, s>>>(sorted, n, dpm);
        if (cudaGetLastError() != cudaSuccess || cudaMemcpyAsync(d_out, dpm, 16, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            st = GZ_ERR_CUDA;
    }
    if (sorted) cudaFreeAsync(sorted, s);
    if (tmp) cudaFreeAsync(tmp, s);
    if (dpm) cudaFreeAsync(dpm, s);
    return st;
}

} // extern "C"
