// nbx_device.cuh -- per-step device math of the spot kernel (sm_100a).
//
// Restates, for the GPU, the loop body of the reference spot kernel
// (/root/reference/pkg/src/xtrace/kernels.py:247-273):
//     h = (rel . a_m) / lambda_w                       kernels.py:253-260
//     F_latt = sincg(pi h, Na) sincg(pi k, Nb) sincg(pi l, Nc)   kernels.py:134-142,261-263
//     F_cell = table[round_half_away(h, k, l)]         kernels.py:145-146,264-268; model.py:264-279
//     acc   += w * (F_cell * F_latt)^2                  kernels.py:269-270
// Design notes:
//   * sin(pi x) is evaluated on the REDUCED argument t = h - n (|t| <= 1/2) and
//     r = N t - rint(N t), so no trigonometric range reduction is ever needed and
//     the grating ratio sin(N pi t)/sin(pi t) becomes (r Q(r^2)) / (t Q(t^2)) with
//     Q(s) = sin(pi sqrt s)/(pi sqrt s) a short even polynomial.  Only |F_latt|^2
//     enters the image, so all signs (-1)^n, (-1)^k drop out.
//   * The reference's limit branch (|sin x| < 1e-12 -> N cos(Nx)/cos(x)) is the
//     t -> 0 limit of the same ratio; biasing |t| by a tiny constant makes the
//     ratio evaluate to N there.  The hot loops skip the bias (t == 0 then gives
//     0/0) and the caller re-runs only a non-finite partial sum with it.
//   * FP32 path: the phase is anchored per (pixel, domain, channel chunk) in
//     FP64 (h0 = S / lambda0 = n0 + f0), and per channel only the small offset
//     x = f0 + S (1/lambda_w - 1/lambda0) is formed in FP32 (|x| <= 2 by the
//     host's chunking), so t carries ~5e-8 absolute error even for |h| ~ 50.
//     All roundings are magic-number adds on the FMA pipe (no FRND/XU).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nbx {

// ---------------------------------------------------------------------------
// Q(s) = sin(pi sqrt(s)) / (pi sqrt(s)), s in [0, 0.2704] (|x| <= 0.52), Q(0) = 1.
// Relative-minimax fits made by tools/fit_sinpi.py (mpmath, 60 digits):
//   FP32 degree 3: max rel err 1.5e-6   (the ratio error stays < 1e-5 per step)
//   FP32 degree 4: max rel err 9.1e-9
//   FP64 degree 6: max rel err 1.2e-13  (1e4 below the 1e-9 parity bar)
//   FP64 degree 7: max rel err 2.9e-16
// ---------------------------------------------------------------------------
template <int V>
constexpr int kDeg = (V == 4) ? 4 : 3;  // Q degree of an FP32 variant (see kMufuNum below)

template <int DEG>
__device__ __forceinline__ float q_sinpi_f32(float s) {
    if constexpr (DEG == 3) {
        float q = -0.1772475662559543266f;
        q = __fmaf_rn(q, s, 0.8095661799590536796f);
        q = __fmaf_rn(q, s, -1.644831841650291668f);
        return __fmaf_rn(q, s, 1.0f);
    } else {
        float q = 0.02460929274903431744f;
        q = __fmaf_rn(q, s, -0.1903951449679496331f);
        q = __fmaf_rn(q, s, 0.8117093632737977162f);
        q = __fmaf_rn(q, s, -1.644933097370079417f);
        return __fmaf_rn(q, s, 1.0f);
    }
}

template <int DEG>
__device__ __forceinline__ double q_sinpi_f64(double s) {
    if constexpr (DEG == 6) {
        double q = 0.0001419369313558917659014215;
        q = __fma_rn(q, s, -0.002343678327814821972139302);
        q = __fma_rn(q, s, 0.02614740711391976615878763);
        q = __fma_rn(q, s, -0.1907517829843114062130668);
        q = __fma_rn(q, s, 0.8117424235039948673634413);
        q = __fma_rn(q, s, -1.64493406682232519873061);
        return __fma_rn(q, s, 1.0);
    } else {
        double q = -0.000006705758238410946132099385;
        q = __fma_rn(q, s, 0.000148310321408001520683082);
        q = __fma_rn(q, s, -0.002346053946710248122556649);
        q = __fma_rn(q, s, 0.02614784439741657402822952);
        q = __fma_rn(q, s, -0.1907518238899222190335658);
        q = __fma_rn(q, s, 0.8117424252758336467922741);
        q = __fma_rn(q, s, -1.644934066848143329530488);
        return __fma_rn(q, s, 1.0);
    }
}

__device__ __forceinline__ float rcp_approx_f32(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// MUFU seed refined by Newton steps (each squares the relative error).
template <int NR>
__device__ __forceinline__ double rcp_f64(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        const double e = __fma_rn(-x, y, 1.0);
        y = __fma_rn(y, e, y);
    }
    return y;
}

// Round half away from zero, exactly as the reference evaluates it:
// floor(x + 0.5) for x >= 0, ceil(x - 0.5) otherwise (kernels.py:145-146).
// trunc(x + copysign(0.5, x)) is the same function bit for bit, including the
// FP rounding of x +- 0.5.
__device__ __forceinline__ double round_half_away(double x) {
    return trunc(x + copysign(0.5, x));
}

// Bias added to |t| so that the grating ratio is finite at exact Bragg
// positions (the reference's limit branch).  Chosen so that the product of
// three biased terms stays a normal number in the path's precision.
constexpr float kTBiasF32 = 1e-12f;
constexpr double kTBiasF64 = 1e-30;
// 1.5 * 2^23: x + kMagicF32 - kMagicF32 == rint(x) for |x| < 2^22, on the FMA pipe.
constexpr float kMagicF32 = 12582912.0f;

// ---------------------------------------------------------------------------
// FP64 axis: numerator r Q(r^2) and denominator t Q(t^2) of |sin(N pi h)/sin(pi h)|,
// plus the reference-rounded index n and t = h - n.
// ---------------------------------------------------------------------------
struct AxisF64 {
    double num, den, n, t;
};

// BIAS = false in the hot loop (|t| used as is; t == 0 gives 0/0, caught by the
// caller), true in the rare re-evaluation that reproduces the limit branch.
template <int DEG, bool BIAS>
__device__ __forceinline__ AxisF64 axis_f64(double S, double iv, double N) {
    AxisF64 a;
    const double h = S * iv;                      // kernels.py:257-260 (sa * (1/lambda))
    a.n = round_half_away(h);                     // lookup index, reference rounding
    a.t = h - a.n;                                // exact (Sterbenz)
    const double ta = BIAS ? fabs(a.t) + kTBiasF64 : fabs(a.t);
    const double k = rint(N * ta);
    const double r = __fma_rn(N, ta, -k);         // N t - k, one rounding
    a.num = r * q_sinpi_f64<DEG>(r * r);
    a.den = ta * q_sinpi_f64<DEG>(ta * ta);
    return a;
}

// ---------------------------------------------------------------------------
// FP32 axis, phase anchored per chunk: x = f0 + S_hi * D where h = n0 + x.
// m = x + M holds j = rint(x) as M + j (used directly by the index FMA chain).
// ---------------------------------------------------------------------------
struct AxisF32 {
    float num, den, j, m, t;
};

// `magic` is kMagicF32 or kMagicF32 + (integer < 2^22): m then carries that
// integer offset for free (the index chain uses it to fold in the chunk's cell).
template <int DEG, bool BIAS>
__device__ __forceinline__ AxisF32 axis_f32(float S_hi, float D, float f0, float N, float magic = kMagicF32) {
    AxisF32 a;
    const float x = __fmaf_rn(S_hi, D, f0);
    a.m = __fadd_rn(x, magic);
    a.j = __fsub_rn(a.m, magic);                  // rint(x), exact
    a.t = __fsub_rn(x, a.j);                      // exact
    const float ta = BIAS ? fabsf(a.t) + kTBiasF32 : fabsf(a.t);
    const float k = __fsub_rn(__fmaf_rn(N, ta, kMagicF32), kMagicF32);  // rint(N t)
    const float r = __fmaf_rn(N, ta, -k);
    a.num = r * q_sinpi_f32<kDeg<DEG>>(r * r);
    a.den = ta * q_sinpi_f32<kDeg<DEG>>(ta * ta);
    return a;
}

// ---------------------------------------------------------------------------
// Non-grating shape transforms, public nanoBragg definitions
// with h0 = round_half_away(h) and fudge = 1:
//   hrad^2 = sum_axes (N t)^2
//   GAUSS : F_latt = NaNbNc exp(-hrad^2 / 0.63)
//   ROUND : F_latt = NaNbNc 0.723601254558268 sinc3(pi sqrt(hrad^2)),
//           sinc3(x) = 3 (sin x / x - cos x) / x^2
//   TOPHAT: F_latt = NaNbNc if hrad^2 < 0.3969 else 0
// Returned as F_latt^2.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T sinc3(T x) {
    if (x < T(1e-4)) {
        // series 1 - x^2/10 avoids the 0/0 cancellation
        return T(1) - x * x * T(0.1);
    }
    T s, c;
    if constexpr (sizeof(T) == 8) {
        sincos(x, &s, &c);
    } else {
        sincosf(x, &s, &c);
    }
    return T(3) * (s / x - c) / (x * x);
}

template <int SHAPE, typename T>
__device__ __forceinline__ T shape_latt2(T hrad2, T nnn) {
    if constexpr (SHAPE == 1) {  // GAUSS
        const T f = nnn * exp(-hrad2 / T(0.63));
        return f * f;
    } else if constexpr (SHAPE == 2) {  // ROUND
        const T f = nnn * T(0.723601254558268) * sinc3<T>(T(3.14159265358979323846) * sqrt(hrad2));
        return f * f;
    } else {  // TOPHAT
        return hrad2 < T(0.3969) ? nnn * nnn : T(0);
    }
}

}  // namespace nbx


namespace nbx {

// ---------------------------------------------------------------------------
// Packed FP32 (sm_100a FFMA2 / FMUL2 / FADD2): two channels per thread in one
// instruction.  The FMA pipe's FLOP rate is unchanged, but every packed op
// takes ONE issue slot for two FMAs, and the FP32 spot loop is issue-bound.
// lo half = channel w, hi half = channel w + 1.  Broadcast operands built with
// bc2() compile to scalar-register operands (R.F32), costing no extra register.
// ---------------------------------------------------------------------------
typedef unsigned long long f2x;

__device__ __forceinline__ f2x pk2(float lo, float hi) {
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f2x bc2(float a) { return pk2(a, a); }
__device__ __forceinline__ float lo2(f2x v) { return __uint_as_float((unsigned)(v & 0xFFFFFFFFull)); }
__device__ __forceinline__ float hi2(f2x v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
    f2x d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
    f2x d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

#ifndef NBX_NUM_MUFU
#define NBX_NUM_MUFU 1  // 0: polynomial numerator on every FP32 variant (the pre-MUFU kernel)
#endif
#ifndef NBX_SIN_LINEAR
#define NBX_SIN_LINEAR 0.0099f
#endif
constexpr float kSinLinear = NBX_SIN_LINEAR;
__device__ __forceinline__ float sin_approx_f32(float x) {
    float y;
    asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int DEG>
__device__ __forceinline__ f2x q_sinpi_f32x2(f2x s) {
    if constexpr (DEG == 3) {
        f2x q = fma2(bc2(-0.1772475662559543266f), s, bc2(0.8095661799590536796f));
        q = fma2(q, s, bc2(-1.644831841650291668f));
        return fma2(q, s, bc2(1.0f));
    } else {
        f2x q = fma2(bc2(0.02460929274903431744f), s, bc2(-0.1903951449679496331f));
        q = fma2(q, s, bc2(0.8117093632737977162f));
        q = fma2(q, s, bc2(-1.644933097370079417f));
        return fma2(q, s, bc2(1.0f));
    }
}

struct AxisF32x2 {
    f2x num, den, j, m;
};

// Numerator of the degree-3 (default) packed path: sin(pi N t) on the XU pipe
// (MUFU.SIN), taking 6 of the 8 FMA-pipe ops of the polynomial form off the
// FMA pipe, which bounds this loop.  MUFU.SIN's absolute error is ~3.4e-7 on
// [-pi, pi] and <= 1.3e-6 up to 10 rad (tools/probes/mix_probe.cu), harmless
// where the numerator is large; near zero its output is fixed-point (~1.6e-7
// absolute), so below |x| = kSinLinear the argument itself is used (relative
// error <= x^2/6 = 1.6e-5; the compiler predicates the MUFU, no select).  The
// numerator is then pi x the polynomial form's (which carries sin(pi r)/pi), so
// a chunk sum is pi^6 times the reference's; domain_sum_f32 rescales it.
// FP32 variants (the DEG template argument of the FP32 helpers):
//   3: degree-3 Q, MUFU numerator (the fast default);
//   4: degree-4 Q, polynomial numerator ("ulp-grade", NBX_FP32_POLY=4);
//   5: degree-3 Q, polynomial numerator (chosen when few samples per pixel would
//      leave MUFU's absolute error un-averaged, e.g. one channel x one domain).
template <int V>
constexpr bool kMufuNum = (V == 3) && (NBX_NUM_MUFU != 0);

// Unbiased (hot-loop) axis for two channels: the same arithmetic as axis_f32
// without |t| (signs drop out of the squared ratio) and without the bias
// (t == 0 -> 0/0 is caught by the caller's finiteness check).  With the MUFU
// numerator N must be passed as pi N.
template <int DEG>
__device__ __forceinline__ AxisF32x2 axis_f32x2(f2x S, f2x D, f2x f0, f2x N, f2x magic) {
    AxisF32x2 a;
    const f2x M = bc2(kMagicF32), neg1 = bc2(-1.0f);
    const f2x x = fma2(S, D, f0);
    a.m = add2(x, magic);
    a.j = fma2(magic, neg1, a.m);         // m - magic = rint(x), exact
    const f2x t = fma2(a.j, neg1, x);     // x - j, exact
    if constexpr (kMufuNum<DEG>) {
        const f2x arg = mul2(N, t);           // pi N t (radians)
        const float a0 = lo2(arg), a1 = hi2(arg);
        const float s0 = fabsf(a0) < kSinLinear ? a0 : sin_approx_f32(a0);
        const float s1 = fabsf(a1) < kSinLinear ? a1 : sin_approx_f32(a1);
        a.num = pk2(s0, s1);
    } else {
        const f2x nk = fma2(fma2(N, t, M), neg1, M);  // -rint(N t)
        const f2x r = fma2(N, t, nk);                 // N t - rint(N t)
        a.num = mul2(r, q_sinpi_f32x2<kDeg<DEG>>(mul2(r, r)));
    }
    a.den = mul2(t, q_sinpi_f32x2<kDeg<DEG>>(mul2(t, t)));
    return a;
}

// Segmented FP32 axis (variant 7): the index j is known per segment, so t = x + (-j) is one
// packed op (exact, as the per-channel x - rint(x)); numerator on MUFU.SIN as above.
__device__ __forceinline__ AxisF32x2 axis_seg_f32x2(f2x S, f2x D, f2x f0, f2x negj, f2x N) {
    AxisF32x2 a;
    const f2x x = fma2(S, D, f0);
    const f2x t = add2(x, negj);
    const f2x arg = mul2(N, t);  // pi N t (radians)
    const float a0 = lo2(arg), a1 = hi2(arg);
    const float s0 = fabsf(a0) < kSinLinear ? a0 : sin_approx_f32(a0);
    const float s1 = fabsf(a1) < kSinLinear ? a1 : sin_approx_f32(a1);
    a.num = pk2(s0, s1);
    a.den = mul2(t, q_sinpi_f32x2<3>(mul2(t, t)));
    a.j = negj;
    a.m = x;
    return a;
}

}  // namespace nbx
