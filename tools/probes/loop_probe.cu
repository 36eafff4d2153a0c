// loop_probe.cu -- FP64 issue-rate probe of the segmented recurrence's channel loop body
// in isolation (no stops, no anchors): is the loop itself FP64-pipe saturated?
//
// Each thread runs the body of domain_sum_f64_cap's uniform loop (six Reinsch sine
// sequences, the two triple products, MUFU.RCP64H + one Newton step, seg += w (nn/dd)^2,
// weight from shared memory) over `iters` channels.  Variants strip one ingredient at a time.
// Prints FP64 warp-instructions per SMSP per cycle (the pipe's ceiling is 0.5: 16 lanes/clk).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o loop_probe loop_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Seq {
    double s, d, a;
};
__device__ __forceinline__ void adv(Seq& q) {
    q.d = __fma_rn(-q.a, q.s, q.d);
    q.s += q.d;
}
__device__ __forceinline__ double rcp1(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = __fma_rn(-x, y, 1.0);
    return __fma_rn(y, e, y);
}

// KIND 0: full body.  1: no MUFU (Newton on a fixed seed).  2: no shared-memory weight.
// 3: 21 independent DFMA chains per channel (pipe ceiling with this occupancy).
// 4: full body + capture selects (the production loop).
template <int KIND, int UNR>
__global__ void __launch_bounds__(128, 6) body(const double* in, double* out, int iters) {
    __shared__ double w[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) w[i] = in[i & 7] * 1e-3 + 1.0;
    __syncthreads();
    const double x = in[8] + threadIdx.x * 1e-5 + blockIdx.x * 1e-7;
    Seq A{0.3 + x, 0.01, 1e-4}, B{0.2 + x, 0.02, 2e-4}, C{0.1 + x, 0.03, 3e-4};
    Seq An{0.6 + x, 0.04, 0.3}, Bn{0.5 + x, 0.05, 0.4}, Cn{0.4 + x, 0.06, 0.5};
    double seg = 0.0, capt = 0.0;
    const int cap = (threadIdx.x * 37) % iters;
    if constexpr (KIND == 3) {
        double r[21];
#pragma unroll
        for (int j = 0; j < 21; ++j) r[j] = x + j;
#pragma unroll UNR
        for (int k = 0; k < iters; ++k) {
#pragma unroll
            for (int j = 0; j < 21; ++j) r[j] = __fma_rn(r[j], 0.999999, 1e-9);
        }
        double s = 0;
#pragma unroll
        for (int j = 0; j < 21; ++j) s += r[j];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
        return;
    }
#pragma unroll UNR
    for (int k = 0; k < iters; ++k) {
        const double wt = KIND == 2 ? 1.000001 : w[k & 255];
        const double nn = (An.s * Bn.s) * Cn.s;
        const double dd = (A.s * B.s) * C.s;
        double y;
        if constexpr (KIND == 1) {
            const double e = __fma_rn(-dd, 0.7, 1.0);
            y = __fma_rn(0.7, e, 0.7);
        } else {
            y = rcp1(dd);
        }
        const double ratio = nn * y;
        if constexpr (KIND == 4) {
            const bool at = k == cap;
            capt = at ? seg : capt;
            seg = __fma_rn(wt, ratio * ratio, at ? 0.0 : seg);
        } else {
            seg = __fma_rn(wt, ratio * ratio, seg);
        }
        adv(A);
        adv(An);
        adv(B);
        adv(Bn);
        adv(C);
        adv(Cn);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = seg + capt + A.s + B.s + C.s + An.s + Bn.s + Cn.s;
}

template <int KIND, int UNR>
void run(const char* name, const double* din, double* dout, int blocks, int iters, double fp64_per_iter) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    body<KIND, UNR><<<blocks, 128>>>(din, dout, iters);
    cudaEventRecord(a);
    body<KIND, UNR><<<blocks, 128>>>(din, dout, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int clk = 0, sms = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double warp_inst = (double)blocks * 4 * iters * fp64_per_iter;
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-34s unroll %d: %8.3f ms  fp64 warp-inst/SMSP/clk %.3f (at %d MHz)\n", name, UNR, ms,
           warp_inst / (sms * 4.0) / cycles, clk / 1000);
}

int main() {
    double h[16];
    for (int i = 0; i < 16; ++i) h[i] = 0.1 * (i + 1);
    double *din, *dout;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 6 * 8;
    cudaMalloc(&din, sizeof(h));
    cudaMalloc(&dout, sizeof(double) * blocks * 128);
    cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
    const int iters = 4096;
    run<0, 4>("full body", din, dout, blocks, iters, 21);
    run<0, 8>("full body", din, dout, blocks, iters, 21);
    run<0, 2>("full body", din, dout, blocks, iters, 21);
    run<4, 4>("full body + capture", din, dout, blocks, iters, 21);
    run<1, 4>("no MUFU", din, dout, blocks, iters, 21);
    run<2, 4>("no LDS weight", din, dout, blocks, iters, 21);
    run<3, 4>("21 independent DFMA chains", din, dout, blocks, iters, 21);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
