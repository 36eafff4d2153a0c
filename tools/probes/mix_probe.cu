// mix_probe.cu -- pipe-concurrency and MUFU.SIN accuracy probes for the FP32 spot loop.
//
// (1) issue/pipe rates on one SM partition: FFMA2 alone, DFMA alone, MUFU.SIN,
//     MUFU.RCP, and FFMA2 + DFMA interleaved at several ratios (do the FMA and
//     FP64 pipes overlap, and at what total issue rate?).
// (2) accuracy of sin.approx.f32 as a function of |x| (relative and absolute),
//     to decide whether the grating NUMERATOR sin(pi N t) may use MUFU.SIN.
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

#define UNROLL 16
typedef unsigned long long f2x;

__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
    f2x d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float sin_approx(float x) {
    float y;
    asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// KIND 0: 8 FFMA2 chains.  1: 8 DFMA chains.  2: 8 MUFU.SIN chains.  3: 8 MUFU.RCP chains.
// 10+R: per unrolled step 8 FFMA2 + R DFMA (independent chains).
template <int KIND>
__global__ void __launch_bounds__(256, 4) probe(double* out, const double* in, int iters, long long* cycles) {
    const double dy = in[0], dz = in[1];
    const float fy = (float)in[0], fz = (float)in[1];
    f2x fx[8], Y, Z;
    double dx[8];
    float sx[8];
    {
        float a = fy, b = fz;
        asm("mov.b64 %0, {%1, %2};" : "=l"(Y) : "f"(a), "f"(a));
        asm("mov.b64 %0, {%1, %2};" : "=l"(Z) : "f"(b), "f"(b));
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float v = 1.0f + threadIdx.x * 1e-7f + c;
        asm("mov.b64 %0, {%1, %2};" : "=l"(fx[c]) : "f"(v), "f"(v));
        dx[c] = v;
        sx[c] = v * 1e-3f;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            if constexpr (KIND == 0) {
#pragma unroll
                for (int c = 0; c < 8; ++c) fx[c] = fma2(fx[c], Y, Z);
            } else if constexpr (KIND == 1) {
#pragma unroll
                for (int c = 0; c < 8; ++c) dx[c] = __fma_rn(dx[c], dy, dz);
            } else if constexpr (KIND == 2) {
#pragma unroll
                for (int c = 0; c < 8; ++c) sx[c] = sin_approx(sx[c]);
            } else if constexpr (KIND == 3) {
#pragma unroll
                for (int c = 0; c < 8; ++c) sx[c] = rcp_approx(sx[c]) + 1.0f;
            } else {
                constexpr int R = KIND - 10;
#pragma unroll
                for (int c = 0; c < 8; ++c) fx[c] = fma2(fx[c], Y, Z);
#pragma unroll
                for (int c = 0; c < R; ++c) dx[c] = __fma_rn(dx[c], dy, dz);
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float a, b;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(fx[c]));
        s += a + b + dx[c] + sx[c];
    }
    if (s == -1.2345) out[0] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, int per_step_warp_instr, double* out, const double* in, long long* cyc, int sms) {
    // 4 blocks x 8 warps per SM (launch bounds guarantee residency): 8 warps per SMSP, one wave
    const int iters = 2000, blocks = sms * 4;
    probe<KIND><<<blocks, 256>>>(out, in, iters / 10, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<KIND><<<blocks, 256>>>(out, in, iters, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    static long long h[8192];
    cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; ++i) mean += h[i];
    mean /= blocks;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double winstr_smsp = (double)iters * UNROLL * per_step_warp_instr * 8;  // per SMSP
    const double clk = ms * 1e-3 * 1.965e9;                                         // SM clocks at 1965 MHz
    printf("%-26s %.3f warp-inst/clk/SMSP by events@1965MHz, %.3f per clock64 tick (ticks/clk %.2f)\n", name,
           winstr_smsp / clk, winstr_smsp / mean, mean / clk);
}

__global__ void sin_acc(const float* x, float* y, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = sin_approx(x[i]);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out, *in;
    long long* cyc;
    cudaMalloc(&out, 16);
    cudaMalloc(&in, 64);
    cudaMalloc(&cyc, sizeof(long long) * 8192);
    double h[8] = {0.99991, 1e-5};
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<0>("FFMA2 x8", 8, out, in, cyc, sms);
    run<1>("DFMA x8", 8, out, in, cyc, sms);
    run<2>("MUFU.SIN x8", 8, out, in, cyc, sms);
    run<3>("MUFU.RCP+FADD x8", 16, out, in, cyc, sms);
    run<11>("FFMA2 x8 + DFMA x1", 9, out, in, cyc, sms);
    run<12>("FFMA2 x8 + DFMA x2", 10, out, in, cyc, sms);
    run<13>("FFMA2 x8 + DFMA x3", 11, out, in, cyc, sms);
    run<14>("FFMA2 x8 + DFMA x4", 12, out, in, cyc, sms);
    run<16>("FFMA2 x8 + DFMA x6", 14, out, in, cyc, sms);
    run<18>("FFMA2 x8 + DFMA x8", 16, out, in, cyc, sms);

    // accuracy of sin.approx.f32 on [-pi, pi]: relative error by decade of |x|, and max abs error
    const int n = 1 << 22;
    float *hx = new float[n], *hy = new float[n];
    for (int i = 0; i < n; ++i) {
        const double u = (double)i / n;  // log-spaced magnitudes 1e-9 .. pi, alternating sign
        hx[i] = (float)((i & 1 ? -1 : 1) * 1e-9 * pow(100.0 / 1e-9, u));
    }
    float *dxp, *dyp;
    cudaMalloc(&dxp, n * 4);
    cudaMalloc(&dyp, n * 4);
    cudaMemcpy(dxp, hx, n * 4, cudaMemcpyHostToDevice);
    sin_acc<<<(n + 255) / 256, 256>>>(dxp, dyp, n);
    cudaMemcpy(hy, dyp, n * 4, cudaMemcpyDeviceToHost);
    double maxabs = 0;
    double rel[12] = {0}, absd[12] = {0};
    for (int i = 0; i < n; ++i) {
        const double want = sin((double)hx[i]);
        const double e = fabs((double)hy[i] - want);
        if (e > maxabs) maxabs = e;
        int dec = (int)floor(log10(fabs((double)hx[i]))) + 9;  // 0 = 1e-9 decade
        if (dec < 0) dec = 0;
        if (dec > 10) dec = 10;
        if (e > absd[dec]) absd[dec] = e;
        const double r = want != 0 ? e / fabs(want) : 0;
        if (r > rel[dec]) rel[dec] = r;
    }
    printf("sin.approx.f32: max abs err %.3e on [-100, 100]\n", maxabs);
    for (int d = 0; d < 11; ++d)
        printf("  |x| in [1e%d, 1e%d): max rel err %.3e  max abs err %.3e\n", d - 9, d - 8, rel[d], absd[d]);
    return 0;
}
