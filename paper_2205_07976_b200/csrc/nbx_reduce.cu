// nbx_reduce.cu -- image statistics and histogram on the device (
// image_stats / image_histogram, /root/reference/pkg/src/xtrace/kernels.py:334-430).
//
// Determinism: like the reference's fixed-tree reduce (execution.py:233-285),
// the summation order depends only on n: block b sums elements
// [b*8192, (b+1)*8192) with a fixed per-thread stride and a fixed shared-memory
// tree, and the per-block partials are combined by one block in a fixed tree.
// min/max are exact; counts are integers (atomics are order-free).
#include <cuda_runtime.h>

#include <cstdint>

namespace nbx {

constexpr int kStatsBlock = 8192;  // kernels.py:343 (_STATS_BLOCK)
constexpr int kThreads = 256;

template <typename T>
__device__ __forceinline__ double load_as_double(const void* p, int64_t i) {
    return (double)static_cast<const T*>(p)[i];
}

struct Partial {
    double mn, mx, sum;
};

__device__ __forceinline__ Partial combine(Partial a, Partial b) {
    return Partial{fmin(a.mn, b.mn), fmax(a.mx, b.mx), a.sum + b.sum};
}

template <typename T>
__global__ void __launch_bounds__(kThreads) stats_blocks_kernel(const void* __restrict__ data, int64_t n,
                                                                Partial* __restrict__ parts) {
    __shared__ Partial sh[kThreads];
    const int64_t lo = (int64_t)blockIdx.x * kStatsBlock;
    const int64_t hi = min(n, lo + kStatsBlock);
    Partial p{INFINITY, -INFINITY, 0.0};
    for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
        const double v = load_as_double<T>(data, i);
        p = combine(p, Partial{v, v, v});
    }
    sh[threadIdx.x] = p;
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = combine(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) parts[blockIdx.x] = sh[0];
}

// One block folds the per-block partials: fixed strided accumulation + fixed tree.
__global__ void __launch_bounds__(kThreads) stats_final_kernel(const Partial* __restrict__ parts, int64_t nb,
                                                               double* __restrict__ out) {
    __shared__ Partial sh[kThreads];
    Partial p{INFINITY, -INFINITY, 0.0};
    for (int64_t i = threadIdx.x; i < nb; i += kThreads) p = combine(p, parts[i]);
    sh[threadIdx.x] = p;
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = combine(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sh[0].mn;
        out[1] = sh[0].mx;
        out[2] = sh[0].sum;
    }
}

// Bin b covers [lo + b w, lo + (b+1) w), the last bin closed above; out-of-range
// values go to underflow / overflow (kernels.py:394-416).  counts has n_bins + 2
// slots: [under, bins..., over]; a shared-memory histogram per block when it fits.
template <typename T>
__global__ void __launch_bounds__(kThreads) histogram_kernel(const void* __restrict__ data, int64_t n, int n_bins,
                                                             double lo, double hi, double width,
                                                             unsigned long long* __restrict__ counts) {
    extern __shared__ unsigned int sh_counts[];
    const bool use_sh = (n_bins + 2) <= 8192;
    if (use_sh)
        for (int i = threadIdx.x; i < n_bins + 2; i += kThreads) sh_counts[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        const double v = load_as_double<T>(data, i);
        int slot;
        if (v < lo) {
            slot = 0;
        } else if (v > hi) {
            slot = n_bins + 1;
        } else {
            int64_t b = (int64_t)floor((v - lo) / width);
            b = b < 0 ? 0 : (b > n_bins - 1 ? n_bins - 1 : b);  // closes the top bin at hi
            slot = (int)b + 1;
        }
        if (use_sh)
            atomicAdd(&sh_counts[slot], 1u);
        else
            atomicAdd(&counts[slot], 1ull);
    }
    __syncthreads();
    if (use_sh)
        for (int i = threadIdx.x; i < n_bins + 2; i += kThreads)
            if (sh_counts[i]) atomicAdd(&counts[i], (unsigned long long)sh_counts[i]);
}

cudaError_t launch_stats(const void* data, int64_t n, int dtype, void* parts, double* out, cudaStream_t st) {
    const int64_t nb = (n + kStatsBlock - 1) / kStatsBlock;
    if (dtype)
        stats_blocks_kernel<double><<<(unsigned)nb, kThreads, 0, st>>>(data, n, static_cast<Partial*>(parts));
    else
        stats_blocks_kernel<float><<<(unsigned)nb, kThreads, 0, st>>>(data, n, static_cast<Partial*>(parts));
    stats_final_kernel<<<1, kThreads, 0, st>>>(static_cast<const Partial*>(parts), nb, out);
    return cudaGetLastError();
}

size_t stats_scratch_bytes(int64_t n) { return sizeof(Partial) * (size_t)((n + kStatsBlock - 1) / kStatsBlock); }

cudaError_t launch_histogram(const void* data, int64_t n, int dtype, int n_bins, double lo, double hi,
                             unsigned long long* counts, cudaStream_t st) {
    const double width = (hi - lo) / n_bins;  // kernels.py:404
    int64_t g = (n + kThreads - 1) / kThreads;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    const size_t smem = (n_bins + 2) <= 8192 ? (size_t)(n_bins + 2) * sizeof(unsigned int) : 0;
    if (dtype)
        histogram_kernel<double><<<(unsigned)g, kThreads, smem, st>>>(data, n, n_bins, lo, hi, width, counts);
    else
        histogram_kernel<float><<<(unsigned)g, kThreads, smem, st>>>(data, n, n_bins, lo, hi, width, counts);
    return cudaGetLastError();
}

}  // namespace nbx
