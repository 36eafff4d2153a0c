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
#pragma once

#include <stdint.h>
#include <math.h>

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
    return NBX_ADD(ldexp((double)m, -53), ldexp(1.0, -54));
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
    return ldexp(p, (int)kf);
}

// log(x) for finite x > 0: x = m 2^e, m in [sqrt(1/2), sqrt(2)), atanh series.
NBX_HD double det_log(double x) {
    int e;
    double m = frexp(x, &e);  // m in [0.5, 1)
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
    if (k < 16.0) {
        double acc = 0.0;
        for (int i = 2; i <= (int)k; ++i) acc = NBX_ADD(acc, det_log((double)i));
        return acc;
    }
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
            p = NBX_MUL(p, mu / k);
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
