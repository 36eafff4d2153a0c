// nbx_poisson.h -- Poisson photon noise shared bit-for-bit by host and device
// (SURVEY §8 X4).  The reference has no noise model, so this
// is builder-defined; parity is "device == host twin, bit-exact".
//
// Bit-exactness rules
//   * Counter-based Philox4x32-10 (Salmon et al., SC'11): key = seed,
//     counter = (pixel lo, pixel hi, image lo ^ image hi, draw#).
//   * Only IEEE-exact operations: + - * / sqrt, floor, ldexp/frexp.  On the
//     device every product/sum goes through __dmul_rn/__dadd_rn, which the
//     compiler never contracts into FMAs; the host side is compiled with
//     -ffp-contract=off.  exp() and log() are written out here (libm and
//     libdevice differ in the last ulp).
//   * Sampler: inversion (sequential search) for mean < 12, Hormann's PTRS
//     transformed rejection (1993) above.
//   * Cheap and divergence-light (a warp's lanes take different branches): log(k!) and
//     1/k from tables of correctly rounded constants, powers of two and frexp from the
//     double's bits (exact, so identical to ldexp / frexp), no per-step division in the
//     inversion search.
#pragma once

#include <stdint.h>
#include <math.h>
#include <string.h>

#if defined(__CUDACC__)
#define NBX_HD __host__ __device__ __forceinline__
#else
#define NBX_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define NBX_MUL(a, b) __dmul_rn((a), (b))
#define NBX_ADD(a, b) __dadd_rn((a), (b))
#define NBX_SUB(a, b) __dsub_rn((a), (b))
#else
#define NBX_MUL(a, b) ((a) * (b))
#define NBX_ADD(a, b) ((a) + (b))
#define NBX_SUB(a, b) ((a) - (b))
#endif

namespace nbx {

// Bit views of a double (exact, both builds).
NBX_HD uint64_t det_bits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, sizeof u);
    return u;
#endif
}
NBX_HD double det_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, sizeof x);
    return x;
#endif
}

// x 2^k, k integral: one exact-product rounding, identical to ldexp; 2^k is built from its bits
// while it is a normal number (k >= -1022), ldexp below.
NBX_HD double det_scale2(double x, int k) {
    if (k >= -1022 && k <= 1023) return NBX_MUL(x, det_from_bits((uint64_t)(k + 1023) << 52));
    return ldexp(x, k);
}

// log(k!) for k < 16, correctly rounded (decimal, 50 digits)
#if defined(__CUDA_ARCH__)
__device__
#endif
static const double kDetLogFact[16] = {
    0.0,
    0.0,
    0.6931471805599453,
    1.791759469228055,
    3.1780538303479458,
    4.787491742782046,
    6.579251212010101,
    8.525161361065415,
    10.60460290274525,
    12.801827480081469,
    15.104412573075516,
    17.502307845873887,
    19.987214495661885,
    22.552163853123425,
    25.19122118273868,
    27.89927138384089};

// 1/k for k <= 64, correctly rounded (IEEE division)
#if defined(__CUDA_ARCH__)
__device__
#endif
static const double kDetInv[65] = {
    0.0,
    1.0,
    0.5,
    0.3333333333333333,
    0.25,
    0.2,
    0.16666666666666666,
    0.14285714285714285,
    0.125,
    0.1111111111111111,
    0.1,
    0.09090909090909091,
    0.08333333333333333,
    0.07692307692307693,
    0.07142857142857142,
    0.06666666666666667,
    0.0625,
    0.058823529411764705,
    0.05555555555555555,
    0.05263157894736842,
    0.05,
    0.047619047619047616,
    0.045454545454545456,
    0.043478260869565216,
    0.041666666666666664,
    0.04,
    0.038461538461538464,
    0.037037037037037035,
    0.03571428571428571,
    0.034482758620689655,
    0.03333333333333333,
    0.03225806451612903,
    0.03125,
    0.030303030303030304,
    0.029411764705882353,
    0.02857142857142857,
    0.027777777777777776,
    0.02702702702702703,
    0.02631578947368421,
    0.02564102564102564,
    0.025,
    0.024390243902439025,
    0.023809523809523808,
    0.023255813953488372,
    0.022727272727272728,
    0.022222222222222223,
    0.021739130434782608,
    0.02127659574468085,
    0.020833333333333332,
    0.02040816326530612,
    0.02,
    0.0196078431372549,
    0.019230769230769232,
    0.018867924528301886,
    0.018518518518518517,
    0.01818181818181818,
    0.017857142857142856,
    0.017543859649122806,
    0.017241379310344827,
    0.01694915254237288,
    0.016666666666666666,
    0.01639344262295082,
    0.016129032258064516,
    0.015873015873015872,
    0.015625};

struct Philox4 {
    uint32_t v[4];
};

NBX_HD void mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
    const uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

NBX_HD Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
        mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    Philox4 out;
    out.v[0] = c0;
    out.v[1] = c1;
    out.v[2] = c2;
    out.v[3] = c3;
    return out;
}

// 53-bit uniform in the open interval (0, 1) from two 32-bit words.
NBX_HD double u53(uint32_t a, uint32_t b) {
    const uint64_t m = ((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6);  // 27 + 26 bits
    return NBX_ADD(NBX_MUL((double)m, 0x1p-53), 0x1p-54);  // exact scalings
}

// exp(x) for x in [-745, 0]: Cody-Waite reduction by ln 2 and a degree-11 Taylor
// polynomial on |r| <= ln2/2 (error < 1 ulp-ish; determinism is what matters).
NBX_HD double det_exp(double x) {
    if (x < -745.0) return 0.0;
    const double ln2_hi = 6.93147180369123816490e-01;
    const double ln2_lo = 1.90821492927058770002e-10;
    const double inv_ln2 = 1.44269504088896338700e+00;
    const double kf = floor(NBX_ADD(NBX_MUL(x, inv_ln2), 0.5));
    const double r = NBX_SUB(NBX_SUB(x, NBX_MUL(kf, ln2_hi)), NBX_MUL(kf, ln2_lo));
    double p = 1.0 / 39916800.0;
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 3628800.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 362880.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 40320.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 5040.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 720.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 120.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 24.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0 / 6.0);
    p = NBX_ADD(NBX_MUL(p, r), 0.5);
    p = NBX_ADD(NBX_MUL(p, r), 1.0);
    p = NBX_ADD(NBX_MUL(p, r), 1.0);
    return det_scale2(p, (int)kf);
}

// log(x) for finite x > 0: x = m 2^e, m in [sqrt(1/2), sqrt(2)), atanh series.
NBX_HD double det_log(double x) {
    int e;
    double m;
    const uint64_t bits = det_bits(x);
    const int ef = (int)((bits >> 52) & 0x7FF);
    if (ef != 0) {  // normal: frexp from the bits (m in [0.5, 1))
        e = ef - 1022;
        m = det_from_bits((bits & 0x800FFFFFFFFFFFFFull) | (1022ull << 52));
    } else {
        m = frexp(x, &e);  // subnormal
    }
    if (m < 0.70710678118654752440) {
        m = NBX_MUL(m, 2.0);
        e -= 1;
    }
    const double f = NBX_SUB(m, 1.0) / NBX_ADD(m, 1.0);
    const double f2 = NBX_MUL(f, f);
    double p = 1.0 / 21.0;
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 19.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 17.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 15.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 13.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 11.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 9.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 7.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 5.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0 / 3.0);
    p = NBX_ADD(NBX_MUL(p, f2), 1.0);
    const double lm = NBX_MUL(NBX_MUL(2.0, f), p);
    const double ed = (double)e;
    return NBX_ADD(NBX_ADD(NBX_MUL(ed, 6.93147180369123816490e-01), lm), NBX_MUL(ed, 1.90821492927058770002e-10));
}

// log(k!) : exact-table for k < 16, Stirling series above.
NBX_HD double det_log_factorial(double k) {
    if (k < 16.0) return kDetLogFact[(int)k];
    const double x = NBX_ADD(k, 1.0);
    const double ix = 1.0 / x;
    const double ix2 = NBX_MUL(ix, ix);
    // 1/(12x) - 1/(360x^3) + 1/(1260x^5) - 1/(1680x^7)
    double s = -1.0 / 1680.0;
    s = NBX_ADD(NBX_MUL(s, ix2), 1.0 / 1260.0);
    s = NBX_ADD(NBX_MUL(s, ix2), -1.0 / 360.0);
    s = NBX_ADD(NBX_MUL(s, ix2), 1.0 / 12.0);
    s = NBX_MUL(s, ix);
    const double half_log_2pi = 0.91893853320467274178;
    return NBX_ADD(NBX_ADD(NBX_SUB(NBX_MUL(NBX_SUB(x, 0.5), det_log(x)), x), half_log_2pi), s);
}

// One Poisson(mu) draw for pixel `pix` of image `image` under `seed`.
NBX_HD double poisson_draw(double mu, uint64_t seed, uint64_t image, uint64_t pix) {
    if (!(mu > 0.0)) return 0.0;        // zero / negative / NaN mean -> 0 counts
    if (mu > 1e15) mu = 1e15;           // keep k representable; far beyond detector counts
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    const uint32_t c0 = (uint32_t)pix, c1 = (uint32_t)(pix >> 32);
    const uint32_t c2 = (uint32_t)image ^ (uint32_t)(image >> 32);
    uint32_t draw = 0;
    if (mu < 12.0) {
        const Philox4 r = philox4x32_10(c0, c1, c2, draw, k0, k1);
        const double u = u53(r.v[0], r.v[1]);
        double p = det_exp(-mu);
        double F = p;
        double k = 0.0;
        while (u > F && k < 1000.0) {
            k = NBX_ADD(k, 1.0);
            const double inv_k = k <= 64.0 ? kDetInv[(int)k] : 1.0 / k;
            p = NBX_MUL(p, NBX_MUL(mu, inv_k));
            F = NBX_ADD(F, p);
        }
        return k;
    }
    const double smu = sqrt(mu);
    const double b = NBX_ADD(0.931, NBX_MUL(2.53, smu));
    const double a = NBX_ADD(-0.059, NBX_MUL(0.02483, b));
    const double inv_alpha = NBX_ADD(1.1239, 1.1328 / NBX_SUB(b, 3.4));
    const double vr = NBX_SUB(0.9277, 3.6224 / NBX_SUB(b, 2.0));
    const double log_mu = det_log(mu);
    for (int it = 0; it < 1000; ++it) {
        const Philox4 r = philox4x32_10(c0, c1, c2, draw++, k0, k1);
        const double U = NBX_SUB(u53(r.v[0], r.v[1]), 0.5);
        const double V = u53(r.v[2], r.v[3]);
        const double us = NBX_SUB(0.5, fabs(U));
        const double k = floor(NBX_ADD(NBX_ADD(NBX_MUL(NBX_ADD(NBX_MUL(2.0, a) / us, b), U), mu), 0.43));
        if (us >= 0.07 && V <= vr) return k;
        if (k < 0.0 || (us < 0.013 && V > us)) continue;
        const double lhs = det_log(NBX_MUL(V, inv_alpha) / NBX_ADD(a / NBX_MUL(us, us), b));
        const double rhs = NBX_SUB(NBX_ADD(-mu, NBX_MUL(k, log_mu)), det_log_factorial(k));
        if (lhs <= rhs) return k;
    }
    return floor(NBX_ADD(mu, 0.5));  // unreachable in practice (acceptance ~0.9/iteration)
}

}  // namespace nbx
