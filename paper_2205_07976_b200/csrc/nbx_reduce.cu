// nbx_reduce.cu -- image statistics and histogram on the device (
// image_stats / image_histogram, /root/reference/pkg/src/xtrace/kernels.py:334-430).
//
// image_stats reproduces the reference's total BIT FOR BIT:
//   * each 8192-pixel block is summed as float(np.sum(chunk, dtype=np.float64))
//     (kernels.py:355-360), i.e. NumPy's pairwise summation of the (exactly
//     upcast) block -- leaves of <= 128 elements with 8 strided accumulators,
//     a power-of-two tree above them, -0.0 start for leaves shorter than 8
//     (numpy/_core/src/umath/loops_utils.h.src, <TYPE>_pairwise_sum; a block
//     fits NumPy's 8192-element cast buffer, so no buffering splits occur);
//   * the block results are combined by parallel_reduce's fixed tree, which
//     splits every span at the largest power of two strictly below its size
//     (execution.py:227-285).
// min/max are exact.  Full blocks are summed by 64 threads (one leaf each, the
// block staged in shared memory); a ragged last block and the cross-block tree
// are evaluated by one thread each with the same recursion.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

namespace nbx {

constexpr int kStatsBlock = 8192;  // kernels.py:343 (_STATS_BLOCK)
constexpr int kThreads = 256;
constexpr int kLeaf = 128;         // NumPy PW_BLOCKSIZE
constexpr int kLeafPad = kLeaf + 1;

template <typename T>
__device__ __forceinline__ double load_as_double(const void* p, int64_t i) {
    return (double)static_cast<const T*>(p)[i];
}

struct Partial {
    double mn, mx, sum;
};

// NumPy's leaf: n < 8 sequential from -0.0; else 8 strided accumulators, a fixed
// tree, then the n % 8 tail sequentially.  `at(i)` reads element i as double.
template <typename F>
__device__ double numpy_leaf(F at, int n) {
    if (n < 8) {
        double res = -0.0;
        for (int i = 0; i < n; ++i) res += at(i);
        return res;
    }
    double r0 = at(0), r1 = at(1), r2 = at(2), r3 = at(3), r4 = at(4), r5 = at(5), r6 = at(6), r7 = at(7);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
        r0 += at(i + 0);
        r1 += at(i + 1);
        r2 += at(i + 2);
        r3 += at(i + 3);
        r4 += at(i + 4);
        r5 += at(i + 5);
        r6 += at(i + 6);
        r7 += at(i + 7);
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res += at(i);
    return res;
}

// NumPy's pairwise recursion (split n/2 rounded down to a multiple of 8), iteratively.
template <typename T>
__device__ double numpy_pairwise(const T* a, int n) {
    struct Frame {
        int off, n, state;
        double left;
    };
    Frame st[16];
    int sp = 0;
    st[0] = Frame{0, n, 0, 0.0};
    double ret = 0.0;
    for (;;) {
        Frame& f = st[sp];
        if (f.n <= kLeaf) {
            const T* b = a + f.off;
            ret = numpy_leaf([b](int i) { return (double)b[i]; }, f.n);
            if (sp == 0) return ret;
            --sp;
            continue;
        }
        int n2 = f.n / 2;
        n2 -= n2 % 8;
        if (f.state == 0) {  // descend left
            f.state = 1;
            st[++sp] = Frame{f.off, n2, 0, 0.0};
        } else if (f.state == 1) {  // left done: descend right
            f.left = ret;
            f.state = 2;
            st[++sp] = Frame{f.off + n2, f.n - n2, 0, 0.0};
        } else {  // right done
            ret = f.left + ret;
            if (sp == 0) return ret;
            --sp;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) stats_blocks_kernel(const void* __restrict__ data, int64_t n,
                                                                Partial* __restrict__ parts) {
    extern __shared__ __align__(16) unsigned char stats_smem[];
    T* blk = reinterpret_cast<T*>(stats_smem);  // 64 leaves of 128 in padded rows (raw T, upcast on use)
    __shared__ double leaf[kStatsBlock / kLeaf];
    __shared__ double mn_s[kThreads / 32], mx_s[kThreads / 32];
    const int64_t lo = (int64_t)blockIdx.x * kStatsBlock;
    const int len = (int)min((int64_t)kStatsBlock, n - lo);
    const T* src = static_cast<const T*>(data) + lo;
    double mn = INFINITY, mx = -INFINITY;
    bool has_nan = false;
    if (len == kStatsBlock) {  // full block: all 32 loads of a thread in flight at once
        constexpr int U = kStatsBlock / kThreads;
        T raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = src[threadIdx.x + kThreads * u];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = threadIdx.x + kThreads * u;
            const double v = (double)raw[u];
            blk[(i / kLeaf) * kLeafPad + (i % kLeaf)] = raw[u];
            mn = fmin(mn, v);
            mx = fmax(mx, v);
            has_nan |= isnan(v);
        }
    } else {
        for (int i = threadIdx.x; i < len; i += kThreads) {  // coalesced staging, exact upcast
            const T raw = src[i];
            const double v = (double)raw;
            blk[(i / kLeaf) * kLeafPad + (i % kLeaf)] = raw;
            mn = fmin(mn, v);
            mx = fmax(mx, v);
            has_nan |= isnan(v);
        }
    }
    // chunk.min() / chunk.max() propagate NaN (NumPy), fmin/fmax skip it (the order of the
    // reduction only matters for the sign of a zero extremum, which the reference leaves unpinned)
    if (__syncthreads_or(has_nan)) mn = mx = NAN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        mn_s[threadIdx.x >> 5] = mn;
        mx_s[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kThreads / 32; ++w) {
            mn_s[0] = fmin(mn_s[0], mn_s[w]);
            mx_s[0] = fmax(mx_s[0], mx_s[w]);
        }
    }
    __syncthreads();
    double sum;
    if (len == kStatsBlock) {
        // pairwise(8192): a perfect binary tree over 64 leaves of 128.  A leaf of 128 is NumPy's
        // 8 strided accumulators r_j = a[j] + a[j + 8] + ... + a[j + 120] (16 terms each, in
        // order), then ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)): lane j of an 8-lane group
        // runs r_j and the group's xor-1, -2, -4 shuffles are that tree (sums commute bit for
        // bit).  A warp's four groups take leaves 8 apart (conflict-free banks on the 129-padded
        // rows); two passes cover the 64 leaves.
        const int j = threadIdx.x & 7, grp = (threadIdx.x >> 3) & 3, w = threadIdx.x >> 5;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
            const int L = w + 8 * grp + 32 * pass;
            const T* row = blk + L * kLeafPad + j;
            double r = (double)row[0];
#pragma unroll
            for (int i = 8; i < kLeaf; i += 8) r += (double)row[i];
            r += __shfl_xor_sync(0xFFFFFFFFu, r, 1);
            r += __shfl_xor_sync(0xFFFFFFFFu, r, 2);
            r += __shfl_xor_sync(0xFFFFFFFFu, r, 4);
            if (j == 0) leaf[L] = r;
        }
        __syncthreads();
        for (int w = kStatsBlock / kLeaf / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) leaf[threadIdx.x] = leaf[2 * threadIdx.x] + leaf[2 * threadIdx.x + 1];
            __syncthreads();
        }
        sum = leaf[0];
    } else {
        sum = threadIdx.x == 0 ? numpy_pairwise<T>(src, len) : 0.0;  // ragged last block
    }
    if (threadIdx.x == 0) parts[blockIdx.x] = Partial{mn_s[0], mx_s[0], 0.0 + sum};
}

// parallel_reduce's tree over the block partials (execution.py:227-285): a span splits
// at the largest power of two strictly below its size.  For nb partials that is the
// binary decomposition of nb into power-of-two segments [s_k, s_k + 2^e_k) (most
// significant first), each reduced as a perfect pairwise tree, then combined right to
// left: T_0 + (T_1 + (... + T_last)).  One block: all segments' tree levels run in
// parallel in place (global scratch, __syncthreads between levels), then thread 0
// folds the chain.
// Python's min(x, y) / max(x, y): y only if it compares below / above x, so a NaN on the
// left survives and one on the right is dropped -- the reference's semantics, NaN included.
__device__ __forceinline__ Partial combine_p(const Partial& x, const Partial& y) {  // kernels.py:362-363
    return Partial{y.mn < x.mn ? y.mn : x.mn, y.mx > x.mx ? y.mx : x.mx, x.sum + y.sum};
}

// The same tree on a copy of the partials in shared memory (nb <= kFinalSmem), one launch-level
// pass instead of a global read-modify-write per level.
constexpr int kFinalSmem = 8192;
__global__ void __launch_bounds__(1024) stats_final_smem_kernel(const Partial* __restrict__ parts_g, int nb,
                                                                double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char final_smem[];
    Partial* parts = reinterpret_cast<Partial*>(final_smem);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) parts[i] = parts_g[i];
    __syncthreads();
    int top = 0;
    while ((1 << (top + 1)) <= nb) ++top;  // highest set bit of nb
    for (int l = 0; l < top; ++l) {
        const int stride = 1 << l;
        for (int q = threadIdx.x; q < nb / (2 * stride); q += blockDim.x) {
            const int i = q * 2 * stride;
            int start = 0, e = top;  // segment of i: nb's set bits, most significant first
            for (; e >= 0; --e) {
                if (!((nb >> e) & 1)) continue;
                if (i < start + (1 << e)) break;
                start += 1 << e;
            }
            if (e > l) parts[i] = combine_p(parts[i], parts[i + stride]);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    int end = nb;
    Partial acc{};
    bool first = true;
    for (int e = 0; e <= top; ++e) {
        if (!((nb >> e) & 1)) continue;
        const int start = end - (1 << e);
        acc = first ? parts[start] : combine_p(parts[start], acc);
        first = false;
        end = start;
    }
    out[0] = acc.mn;
    out[1] = acc.mx;
    out[2] = acc.sum;
}

__global__ void __launch_bounds__(1024) stats_final_kernel(Partial* __restrict__ parts, int64_t nb,
                                                           double* __restrict__ out) {
    int top = 0;
    while ((int64_t(1) << (top + 1)) <= nb) ++top;  // highest set bit of nb
    for (int l = 0; l < top; ++l) {
        const int64_t stride = int64_t(1) << l;
        // pair (i, i + stride) for i a multiple of 2 stride inside any segment longer than 2 stride
        for (int64_t q = threadIdx.x; q < nb / (2 * stride); q += blockDim.x) {
            const int64_t i = q * 2 * stride;
            // segment of i: the prefix of nb's set bits (most significant first) that contains i
            int64_t start = 0;
            int e = top;
            for (; e >= 0; --e) {
                if (!((nb >> e) & 1)) continue;
                if (i < start + (int64_t(1) << e)) break;
                start += int64_t(1) << e;
            }
            if (e > l) parts[i] = combine_p(parts[i], parts[i + stride]);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    // segment roots, least significant (rightmost) first: acc = T_k + acc
    int64_t end = nb;
    Partial acc{};
    bool first = true;
    for (int e = 0; e <= top; ++e) {
        if (!((nb >> e) & 1)) continue;
        const int64_t start = end - (int64_t(1) << e);
        acc = first ? parts[start] : combine_p(parts[start], acc);
        first = false;
        end = start;
    }
    out[0] = acc.mn;
    out[1] = acc.mx;
    out[2] = acc.sum;
}

// Bin b covers [lo + b w, lo + (b+1) w), the last bin closed above; out-of-range
// values go to underflow / overflow (kernels.py:394-416).  counts has n_bins + 2
// slots: [under, bins..., over]; a shared-memory histogram per warp (or per block, or
// global atomics) when it fits.
//
// The bin is the reference's floor((v - lo) / width) (kernels.py:409) without an FP64
// division per element: q = (v - lo) * RN(1 / width) is within 3.3e-16 q of the
// correctly rounded quotient, so the two floors can differ only when an integer lies
// within that distance of q -- then (and for NaN) the exact division decides.
__device__ __forceinline__ int hist_slot(double v, int n_bins, double lo, double hi, double width, double inv_w) {
    if (v < lo) return 0;
    if (v > hi) return n_bins + 1;
    const double d = v - lo;
    const double q = d * inv_w;
    const double fq = floor(q);
    const double f = q - fq;                 // exact below 2^52
    const double m = q * 1e-15;              // 3x the bound above
    int64_t b;
    if (f > m && f < 1.0 - m)
        b = (int64_t)fq;
    else
        b = (int64_t)floor(d / width);      // kernels.py:409, NaN included
    b = b < 0 ? 0 : (b > n_bins - 1 ? n_bins - 1 : b);  // closes the top bin at hi
    return (int)b + 1;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) histogram_kernel(const void* __restrict__ data, int64_t n, int n_bins,
                                                             double lo, double hi, double width, double inv_w,
                                                             unsigned long long* __restrict__ counts) {
    extern __shared__ unsigned int sh_counts[];
    const int slots = n_bins + 2;
    const int warp_hists = slots * (kThreads / 32) <= 8192 ? kThreads / 32 : 1;  // private per warp when small
    const bool use_sh = slots <= 8192;
    if (use_sh)
        for (int i = threadIdx.x; i < slots * warp_hists; i += kThreads) sh_counts[i] = 0;
    __syncthreads();
    unsigned int* my = sh_counts + (warp_hists > 1 ? (threadIdx.x / 32) * slots : 0);
    auto add = [&](double v) {
        const int slot = hist_slot(v, n_bins, lo, hi, width, inv_w);
        if (use_sh)
            atomicAdd(&my[slot], 1u);
        else
            atomicAdd(&counts[slot], 1ull);
    };
    const T* p = static_cast<const T*>(data);
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte load
    const int64_t nv = (reinterpret_cast<uintptr_t>(p) & 15) == 0 ? n / V : 0;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    const int64_t t0 = blockIdx.x * (int64_t)kThreads + threadIdx.x;
    using V4 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    const V4* pv = reinterpret_cast<const V4*>(p);
    auto add_v = [&](const V4& q) {
        if constexpr (sizeof(T) == 4) {
            add(q.x), add(q.y), add(q.z), add(q.w);
        } else {
            add(q.x), add(q.y);
        }
    };
    constexpr int kInFlight = 4;  // loads issued before their values are binned (memory-level parallelism)
    int64_t i = t0;
    for (; i + (kInFlight - 1) * stride < nv; i += kInFlight * stride) {
        V4 q[kInFlight];
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) q[u] = pv[i + u * stride];
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) add_v(q[u]);
    }
    for (; i < nv; i += stride) add_v(pv[i]);
    for (int64_t i = nv * V + t0; i < n; i += stride) add((double)p[i]);
    __syncthreads();
    if (use_sh)
        for (int i = threadIdx.x; i < slots; i += kThreads) {
            unsigned long long c = 0;
            for (int w = 0; w < warp_hists; ++w) c += sh_counts[w * slots + i];
            if (c) atomicAdd(&counts[i], c);
        }
}

cudaError_t launch_stats(const void* data, int64_t n, int dtype, void* parts, double* out, cudaStream_t st) {
    const int64_t nb = (n + kStatsBlock - 1) / kStatsBlock;
    const int rows = kStatsBlock / kLeaf * kLeafPad;
    if (dtype) {
        const size_t smem = (size_t)rows * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(stats_blocks_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        stats_blocks_kernel<double><<<(unsigned)nb, kThreads, smem, st>>>(data, n, static_cast<Partial*>(parts));
    } else {
        const size_t smem = (size_t)rows * sizeof(float);
        stats_blocks_kernel<float><<<(unsigned)nb, kThreads, smem, st>>>(data, n, static_cast<Partial*>(parts));
    }
    if (nb <= kFinalSmem) {
        const size_t smem = sizeof(Partial) * (size_t)nb;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(stats_final_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
        }
        stats_final_smem_kernel<<<1, 1024, smem, st>>>(static_cast<const Partial*>(parts), (int)nb, out);
    } else {
        stats_final_kernel<<<1, 1024, 0, st>>>(static_cast<Partial*>(parts), nb, out);
    }
    return cudaGetLastError();
}

size_t stats_scratch_bytes(int64_t n) { return sizeof(Partial) * (size_t)((n + kStatsBlock - 1) / kStatsBlock); }

cudaError_t launch_histogram(const void* data, int64_t n, int dtype, int n_bins, double lo, double hi,
                             unsigned long long* counts, cudaStream_t st) {
    const double width = (hi - lo) / n_bins;  // kernels.py:404
    const double inv_w = 1.0 / width;
    int64_t g = (n + 4 * kThreads - 1) / (4 * kThreads);
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    const int slots = n_bins + 2;
    const int warp_hists = slots * (kThreads / 32) <= 8192 ? kThreads / 32 : 1;
    const size_t smem = slots <= 8192 ? (size_t)slots * warp_hists * sizeof(unsigned int) : 0;
    if (dtype)
        histogram_kernel<double><<<(unsigned)g, kThreads, smem, st>>>(data, n, n_bins, lo, hi, width, inv_w, counts);
    else
        histogram_kernel<float><<<(unsigned)g, kThreads, smem, st>>>(data, n, n_bins, lo, hi, width, inv_w, counts);
    return cudaGetLastError();
}

}  // namespace nbx
