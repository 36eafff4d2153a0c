// pipe_probe.cu -- issue-rate microbenchmarks for the FP32 instruction forms the
// spot kernel uses (3-register FFMA vs immediate-operand FFMA, FMUL, FADD, mixes).
// Reports warp-instructions per cycle per SM partition (SMSP) from clock64().
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
#define UNROLL 16

template <int KIND>
__global__ void __launch_bounds__(512) probe(float* out, const float* in, int iters, long long* cycles) {
    float y = in[0], z = in[1];  // runtime values: the compiler cannot make them immediates
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = in[2 + c] + threadIdx.x * 1e-7f;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) {
                if (KIND == 0) x[c] = __fmaf_rn(x[c], y, z);                 // FFMA R,R,R
                if (KIND == 1) x[c] = __fmaf_rn(x[c], 0.99991f, 1e-5f);     // FFMA R,imm,imm
                if (KIND == 2) x[c] = __fmul_rn(x[c], y);                   // FMUL R,R
                if (KIND == 3) x[c] = __fadd_rn(x[c], 1e-5f);               // FADD R,imm
                if (KIND == 4) x[c] = (c & 1) ? __fmaf_rn(x[c], y, z) : __fmaf_rn(x[c], 0.99991f, 1e-5f);
                if (KIND == 5) x[c] = __fadd_rn(x[c], y);                   // FADD R,R
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == -1.2345f) out[0] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, float* out, const float* in, long long* cyc, int sms) {
    const int iters = 2000, blocks = sms * 4;
    probe<KIND><<<blocks, 512>>>(out, in, iters / 10, cyc);
    probe<KIND><<<blocks, 512>>>(out, in, iters, cyc);
    cudaDeviceSynchronize();
    long long h[4096];
    cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; ++i) mean += h[i];
    mean /= blocks;
    // 4 blocks x 16 warps resident per SM, 4 SMSPs: warp-instr per SMSP per cycle
    const double winstr = (double)iters * UNROLL * CHAINS * 16 * 4 / 4;
    printf("%-28s %.3f warp-inst/clk/SMSP\n", name, winstr / mean);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out, *in;
    long long* cyc;
    cudaMalloc(&out, 16);
    cudaMalloc(&in, 64);
    cudaMalloc(&cyc, sizeof(long long) * 4096);
    float h[16] = {0.99991f, 1e-5f, 1, 2, 3, 4, 5, 6, 7, 8};
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<0>("FFMA R,R,R", out, in, cyc, sms);
    run<1>("FFMA R,imm,imm", out, in, cyc, sms);
    run<2>("FMUL R,R", out, in, cyc, sms);
    run<3>("FADD R,imm", out, in, cyc, sms);
    run<4>("FFMA 50/50 reg/imm", out, in, cyc, sms);
    run<5>("FADD R,R", out, in, cyc, sms);
    return 0;
}
